"""Per-kernel share of an ncu launch list (--metrics gpu__time_duration.sum --csv).

  python tools/launch_summary.py gpurun_out/launches.csv > profiles/rNN_launches.md
ncu's per-launch times are cold-cache and serialised: compare SHARES, not absolutes.
"""
import collections
import csv
import sys


def main(path):
    lines = [ln for ln in open(path) if ln.startswith('"')]
    rows = list(csv.reader(lines))
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot = collections.defaultdict(lambda: [0, 0.0])
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}
    for r in rows[1:]:
        name = r[ki].split("(")[0]
        tot[name][0] += 1
        tot[name][1] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-6)
    T = sum(v[1] for v in tot.values())
    print(f"ncu launch list `{path}`: {sum(v[0] for v in tot.values())} launches, {T:.1f} ms serialised\n")
    print("| kernel | launches | total ms | ms/launch | share |")
    print("|---|---|---|---|---|")
    for n, (c, t) in sorted(tot.items(), key=lambda x: -x[1][1]):
        print(f"| `{n}` | {c} | {t:.2f} | {t / c:.3f} | {100 * t / T:.2f}% |")


if __name__ == "__main__":
    main(sys.argv[1])

"""Warp-stall samples of an ncu --set full report by site: the mbarrier wait loops
(the sample lands on the branch after SYNCS ... TRYWAIT), the TMA issue, and the rest,
split by warp role from the code layout (producer = around the UTMALDG block).
  python tools/stall_sites.py gpurun_out/c4prof_....ncu-rep"""
import csv
import io
import subprocess
import sys


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    data = []
    for r in rows[2:]:
        if len(r) != len(hdr) or not r[0].startswith("0x"):
            if data:
                break
            continue
        data.append(r)
    return hdr, data


def main(rep):
    hdr, data = load(rep)
    ix = {h: i for i, h in enumerate(hdr)}
    S = ix["Warp Stall Sampling (All Samples)"]
    E = ix["Instructions Executed"]
    tot = sum(int(r[S]) for r in data)
    print(f"{rep}: {tot} samples, {len(data)} SASS instructions")
    for i, r in enumerate(data):
        if "TRYWAIT" in r[1] and i + 1 < len(data):
            # (the branch back to the retry loop may follow a few instructions later)
            j = next((j for j in range(i + 1, min(i + 5, len(data))) if "BRA" in data[j][1]), i + 1)
            n = sum(int(data[t][S]) for t in range(i, j + 1))
            if n > 0.005 * tot:
                bar = r[1].split("[")[1].split("]")[0]
                print(f"  wait {r[0][-5:]} [{bar}] {n:8d} {100 * n / tot:5.1f} %  execs {r[E]}")
    tma = [i for i, r in enumerate(data) if "UTMALDG" in r[1]]
    if tma:
        a, b = max(0, tma[0] - 30), tma[-1] + 5
        n = sum(int(data[i][S]) for i in range(a, b))
        print(f"  producer block (incl. its waits) {n:8d} {100 * n / tot:5.1f} %")
    cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    agg = {c[6:]: sum(int(r[ix[c]]) for r in data) for c in cols}
    print("  reasons:", ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))


if __name__ == "__main__":
    for rep in sys.argv[1:]:
        main(rep)

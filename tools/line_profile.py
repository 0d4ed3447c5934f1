"""Per-source-line executed instructions / stall samples / branch share of one ncu capture.

  python tools/line_profile.py gpurun_out/x.ncu-rep [N]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def f(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return 0.0


def main(path, n=30):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    agg = defaultdict(lambda: [0.0, 0.0, 0.0, ""])
    ops = defaultdict(float)
    fname = h = line = None
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Function Name":
            continue
        if r[0] == "Line No":
            h = r
            iss = h.index("Warp Stall Sampling (All Samples)")
            iex = h.index("Instructions Executed")
            continue
        if r[0]:
            line = (fname, int(r[0]))
            agg[line][3] = r[1].strip()[:80]
        if h and len(r) > iex and r[3]:
            o = r[3].split()
            if not o:
                continue
            o = o[1] if o[0].startswith("@") and len(o) > 1 else o[0]
            agg[line][0] += f(r[iss])
            agg[line][1] += f(r[iex])
            ops[o.split(".")[0]] += f(r[iex])
            if o.startswith("BRA"):
                agg[line][2] += f(r[iex])
    tot = sum(v[0] for v in agg.values()) or 1
    te = sum(v[1] for v in agg.values()) or 1
    print(f"{path}: {te:.4g} warp instructions")
    print("opcodes:", ", ".join(f"{k} {100 * v / te:.1f}%" for k, v in sorted(ops.items(), key=lambda x: -x[1])[:14]))
    for l, (s, e, b, src) in sorted(agg.items(), key=lambda x: -x[1][1])[:n]:
        print(f"{l[0][:14]}:{l[1]:4d} samp {100 * s / tot:5.1f}% exec {100 * e / te:5.1f}% bra {100 * b / te:4.1f}%  {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)

"""DRAM traffic per cell of the hot kernels from `ncu --set full` captures.

  python tools/make_traffic.py [--cells N] gpurun_out/prof_*.ncu-rep > profiles/ncu_traffic.json

The captures come from tools/prof_kernels.sh (tools/profile_step.py: the c4 recipe
at the c3 size 256 x 256 x 512, one launch per kernel; --cells 268435456 for captures
of the full c4 grid).  bench.py multiplies the per-cell figure by its local cell count
to fill roofline.traffic.
"""
import csv
import io
import json
import re
import subprocess
import sys

CELLS = 256 * 256 * 512
# demangled kernel name -> bench.py kernel class
CLASSES = [
    (r"^void (sts::)?aniso_tma_kernel<(\(int\))?2,", "aniso_rkl2_stage"),
    (r"^void aniso_tma_kernel<5,", "aniso_pcg_s"),
    (r"^void iso_tma_kernel<2,", "iso_rkl2_stage"),
    (r"^void iso_tma_kernel<5,", "iso_pcg_s"),
    (r"^void aniso_tma_kernel<6,", "aniso_pcg_m"),
    (r"^void aniso_tma_kernel<7,", "aniso_rkl2_dstage"),
    (r"^void iso_tma_kernel<7,", "iso_rkl2_dstage"),
    (r"^void iso_tma_kernel<6,", "iso_pcg_m"),
    (r"^void pcg_rupdate_kernel<3>", "pcg_update_c3"),
    (r"^void pcg_rupdate_kernel<1>", "pcg_update"),
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main(paths, cells=CELLS):
    out = {"cells": cells, "source": "ncu --set full --clock-control none, tools/prof_kernels.sh",
           "dram_bytes_per_cell": {}, "dram_pct": {}, "duration_us": {}}
    acc = {}   # class -> [(bytes/cell, dram %, us)] over the captured launches (averaged: the merged
    #            PCG passes alternate a skipped and a catch-up x update)
    for p in paths:
        txt = subprocess.run(["ncu", "-i", p, "--page", "raw", "--csv"],
                             capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(txt)))
        if len(rows) < 3:
            continue
        h, u = rows[0], rows[1]
        for r in rows[2:]:
            d = dict(zip(h, r))
            name = d.get("Kernel Name", "")
            cls = next((c for pat, c in CLASSES if re.search(pat, name)), None)
            if cls is None:
                continue
            rd = float(d["dram__bytes_read.sum"].replace(",", "")) * SCALE[u[h.index("dram__bytes_read.sum")]]
            wr = float(d["dram__bytes_write.sum"].replace(",", "")) * SCALE[u[h.index("dram__bytes_write.sum")]]
            pct = float(d["gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"].replace(",", ""))
            dur = float(d["gpu__time_duration.sum"].replace(",", ""))
            unit = u[h.index("gpu__time_duration.sum")]
            acc.setdefault(cls, []).append(((rd + wr) / cells, pct, dur * {"ns": 1e-3, "us": 1.0, "ms": 1e3}.get(unit, 1.0)))
    for cls, v in acc.items():
        out["dram_bytes_per_cell"][cls] = round(sum(x[0] for x in v) / len(v), 3)
        out["dram_pct"][cls] = round(sum(x[1] for x in v) / len(v), 3)
        out["duration_us"][cls] = round(sum(x[2] for x in v) / len(v), 3)
        out.setdefault("launches_averaged", {})[cls] = len(v)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    args = sys.argv[1:]
    cells = CELLS
    if args and args[0] == "--cells":
        cells, args = int(args[1]), args[2:]
    main(args, cells)

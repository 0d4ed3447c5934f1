"""Summarise tools/ab_ncu.sh output: per variant and kernel, ms and DRAM B/cell."""
import csv
import glob
import io
import sys

CELLS = float(sys.argv[1]) if len(sys.argv) > 1 and not sys.argv[1].endswith(".csv") else 268435456.0
for f in sorted(glob.glob("gpurun_out/abncu_*.csv")):
    lines = [ln for ln in open(f) if ln.startswith('"')]
    if not lines:
        print(f, "no data")
        continue
    rows = list(csv.reader(io.StringIO("".join(lines))))
    h = rows[0]
    mi, vi, ui = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    vals = {}
    for r in rows[1:]:
        v = float(r[vi].replace(",", ""))
        u = r[ui]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "usecond": 1e-3,
                 "msecond": 1.0, "ns": 1e-6, "us": 1e-3, "ms": 1.0}.get(u, 1.0)
        vals.setdefault(r[mi], []).append(v * scale)
    avg = {k: sum(v) / len(v) for k, v in vals.items()}
    rd, wr = avg.get("dram__bytes_read.sum", 0), avg.get("dram__bytes_write.sum", 0)
    print(f"{f.split('abncu_')[1][:-4]:45s} {avg.get('gpu__time_duration.sum', 0):8.3f} ms  "
          f"DRAM {rd / CELLS:6.1f} + {wr / CELLS:5.1f} B/cell  L2 hit {avg.get('lts__t_sector_hit_rate.pct', 0):5.1f}%  "
          f"clk {avg.get('sm__cycles_elapsed.avg.per_second', 0) / 1e9:5.2f} GHz")

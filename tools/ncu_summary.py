"""Summarise ncu --set full reports (.ncu-rep) into a markdown table + JSON.

  python tools/ncu_summary.py gpurun_out/prof_*.ncu-rep > profiles/rNN_ncu_summary.md
"""
import csv
import io
import json
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_active": "l1_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "smsp__inst_executed.sum": "inst",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pct",
    "smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio": "stall_long_sb",
}


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for i, h in enumerate(hdr):
            if h in WANT or h == "Kernel Name":
                d[WANT.get(h, "kernel")] = (r[i], units[i])
        res.append(d)
    return res


def stall_reasons(path, top=6):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    hdr = rows[0]
    vals = rows[2]
    st = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            try:
                st.append((float(vals[i].replace(",", "")),
                           h.split("stalled_")[1].replace("_per_issue_active.ratio", "")))
            except ValueError:
                pass
    return [f"{n}:{v:.2f}" for v, n in sorted(st, reverse=True)[:top]]


def main(paths):
    allres = {}
    print("| kernel | dur | DRAM rd+wr / launch | DRAM % | SM % | L1 % | L2 hit | occ % | regs | FP64 % | top stalls |")
    print("|---|---|---|---|---|---|---|---|---|---|---|")
    for p in paths:
        for d in raw(p):
            g = lambda k: d.get(k, ("", ""))[0]  # noqa: E731
            name = g("kernel")[:60]
            try:
                rd = float(g("dram_read").replace(",", ""))
                wr = float(g("dram_write").replace(",", ""))
                sc = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
                tot = rd * sc.get(d["dram_read"][1], 1) + wr * sc.get(d["dram_write"][1], 1)
            except Exception:
                tot = float("nan")
            st = stall_reasons(p)
            allres[p] = {"kernel": name, "dram_bytes": tot, **{k: g(k) for k in WANT.values()}, "stalls": st}
            print(f"| {name} | {g('duration')} {d.get('duration', ('', ''))[1]} | {tot / 1e9:.3f} GB | {g('dram_pct')} | "
                  f"{g('sm_pct')} | {g('l1_pct')} | {g('l2_hit')} | {g('occupancy')} | {g('regs')} | {g('fp64_pct')} | "
                  f"{' '.join(st)} |")
    print()
    print("```json")
    print(json.dumps(allres, indent=1))
    print("```")


if __name__ == "__main__":
    main(sys.argv[1:])

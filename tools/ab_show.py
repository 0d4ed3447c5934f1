"""Print the A-B bench lines of gpurun_out/ab_*.log (value, hot-kernel fractions / ms)."""
import glob
import json

for f in sorted(glob.glob("gpurun_out/ab_*.log")):
    for ln in open(f):
        if ln.startswith("{"):
            d = json.loads(ln)
            k = d["kernels"]
            print(f.split("/")[-1], round(d["value"], 3),
                  {n: (k[n]["frac"], round(k[n]["ms"], 1)) for n in
                   ("iso_pcg_m", "aniso_pcg_m", "iso_rkl2_dstage", "aniso_rkl2_dstage", "aniso_gersh", "face_kappa")
                   if n in k}, d["clocks"]["sm_mhz"])

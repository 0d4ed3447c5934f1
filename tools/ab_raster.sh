# A-B of the CTA rasterisation: the product build (theta-first bands of
# 8 tiles) against the plain 3-D grid order, same bench command, back to back.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python paper_1610_01265_b200/build.py -DANISO_RASTER_H=0 -DISO_RASTER_H=0 \
    --out=paper_1610_01265_b200/libsts_b200_r0.so > gpurun_out/build_r0.log 2>&1
for v in r0 prod r0 prod; do
  if [ $v = r0 ]; then export STS_LIB=$PWD/paper_1610_01265_b200/libsts_b200_r0.so; else unset STS_LIB; fi
  timeout 600 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ab_$v.log 2>&1
  python - <<PY
import json
for ln in open("gpurun_out/ab_$v.log"):
    if ln.startswith("{"):
        d = json.loads(ln); k = d["kernels"]
        print("$v", round(d["value"], 3), {n: k[n]["frac"] for n in ("iso_pcg_m", "aniso_pcg_m", "iso_rkl2_dstage", "aniso_rkl2_dstage")}, d["clocks"]["sm_mhz"])
PY
done

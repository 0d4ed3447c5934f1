# DRAM bytes (ncu) and bench of raster band heights 2 and 4 against the product (0)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for H in 2 4; do
  python paper_1610_01265_b200/build.py -DANISO_RASTER_H=$H -DISO_RASTER_H=$H \
      --out=paper_1610_01265_b200/libsts_b200_h$H.so > gpurun_out/build_h$H.log 2>&1
done
VARIANTS="h0= h2=paper_1610_01265_b200/libsts_b200_h2.so h4=paper_1610_01265_b200/libsts_b200_h4.so" bash tools/ab_ncu.sh > gpurun_out/ab_ncu.log 2>&1
python tools/ab_ncu_summary.py
for v in h2 h0 h4 h0; do
  if [ $v = h0 ]; then unset STS_LIB; else export STS_LIB=$PWD/paper_1610_01265_b200/libsts_b200_$v.so; fi
  timeout 600 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ab_$v.log 2>&1
  python - <<PY
import json
for ln in open("gpurun_out/ab_$v.log"):
    if ln.startswith("{"):
        d = json.loads(ln); k = d["kernels"]
        print("$v", round(d["value"], 3), {n: (k[n]["frac"], k[n]["ms"]) for n in ("iso_pcg_m", "aniso_pcg_m", "iso_rkl2_dstage", "aniso_rkl2_dstage") if n in k}, d["clocks"]["sm_mhz"])
PY
done

# A-B of a compile-time knob on the default bench (same box, alternating runs).
#   VDEFS="-DANISO_M_DREAD=1" bash tools/ab_bench.sh
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python paper_1610_01265_b200/build.py $VDEFS --out=paper_1610_01265_b200/libsts_b200_v.so > gpurun_out/build_v.log 2>&1
for v in v prod v prod; do
  if [ $v = v ]; then export STS_LIB=$PWD/paper_1610_01265_b200/libsts_b200_v.so; else unset STS_LIB; fi
  timeout 600 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline ${BARGS:-} > gpurun_out/ab_$v.log 2>&1
  python - <<PY
import json
for ln in open("gpurun_out/ab_$v.log"):
    if ln.startswith("{"):
        d = json.loads(ln); k = d["kernels"]
        print("$v", round(d["value"], 3), {n: (k[n]["frac"], k[n]["ms"]) for n in ("iso_pcg_m", "aniso_pcg_m", "iso_rkl2_dstage", "aniso_rkl2_dstage") if n in k}, d["clocks"]["sm_mhz"])
PY
done

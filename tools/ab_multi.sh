# A-B of several compile-time variants on the default bench (same box, interleaved).
#   VARIANTS="a:-DX=1 b:-DY=2" bash tools/ab_multi.sh
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for pair in $VARIANTS; do
  name=${pair%%:*}; defs=${pair#*:}
  python paper_1610_01265_b200/build.py $(echo $defs | tr ',' ' ') --out=paper_1610_01265_b200/libsts_b200_$name.so > gpurun_out/build_$name.log 2>&1
done
for round in 1 2; do
  for v in prod $(for pair in $VARIANTS; do echo ${pair%%:*}; done); do
    if [ $v = prod ]; then unset STS_LIB; else export STS_LIB=$PWD/paper_1610_01265_b200/libsts_b200_$v.so; fi
    timeout 600 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline ${BARGS:-} > gpurun_out/ab_$v.log 2>&1
    python - <<PY
import json
for ln in open("gpurun_out/ab_$v.log"):
    if ln.startswith("{"):
        d = json.loads(ln); k = d["kernels"]
        print("$v", round(d["value"], 3), {n: (k[n]["frac"], k[n]["ms"]) for n in ("iso_pcg_m", "aniso_pcg_m", "iso_rkl2_dstage", "aniso_rkl2_dstage") if n in k}, d["clocks"]["sm_mhz"])
PY
  done
done

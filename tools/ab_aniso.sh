# A-B of anisotropic tile variants: parity tests of each variant, then the c3 bench
# (conduction only) and the c4 bench, interleaved on the same box.
#   VARIANTS="old:-DANISO_RB=1,-DANISO_NW=8 r3:-DANISO_RB=3,-DANISO_M_MINB=2,-DANISO_MINB=2" bash tools/ab_aniso.sh
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for pair in $VARIANTS; do
  name=${pair%%:*}; defs=${pair#*:}
  [ "$defs" = prebuilt ] && continue   # (built here from another tree, shipped in the snapshot)
  python paper_1610_01265_b200/build.py $(echo $defs | tr ',' ' ') --out=paper_1610_01265_b200/libsts_b200_$name.so > gpurun_out/build_$name.log 2>&1 || exit 1
done
names="prod $(for pair in $VARIANTS; do echo ${pair%%:*}; done)"
for v in $names; do
  if [ $v = prod ]; then unset STS_LIB; else export STS_LIB=$PWD/paper_1610_01265_b200/libsts_b200_$v.so; fi
  timeout 600 python -m pytest tests -m gpu -x -q -k "${TESTK:-tma_kernels_match or spitzer or be_pcg or aniso or virtual or graph}" > gpurun_out/abt_$v.log 2>&1
  echo "$v tests: $(tail -1 gpurun_out/abt_$v.log)"
done
for cfg in ${CFGS:-c3_spitzer256 c4_scale512}; do
for round in 1 2; do
  for v in $names; do
    if [ $v = prod ]; then unset STS_LIB; else export STS_LIB=$PWD/paper_1610_01265_b200/libsts_b200_$v.so; fi
    timeout 600 python bench.py --config $cfg --steps ${STEPS:-5} --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ab_${cfg}_$v.log 2>&1
    python - <<PY
import json
for ln in open("gpurun_out/ab_${cfg}_$v.log"):
    if ln.startswith("{"):
        d = json.loads(ln); k = d["kernels"]
        print("$cfg $v", round(d["value"], 3), {n: (k[n]["frac"], round(k[n]["ms"], 1)) for n in ("iso_pcg_m", "aniso_pcg_m", "iso_rkl2_dstage", "aniso_rkl2_dstage", "aniso_gersh") if n in k}, d["clocks"]["sm_mhz"])
PY
  done
done
done

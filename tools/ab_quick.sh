# Quick A-B on one box: build the product and the variants, parity tests of each
# (tests/test_gpu_parity.py only, filtered by TESTK), ONE interleaved round of the bench
# on CFGS (default c3), then optional ncu captures of the product (KERNELS, see
# tools/prof_kernels.sh).
#   VARIANTS="r3:-DANISO_RB=3,-DANISO_MINB=2 old:prebuilt" CFGS="c3_spitzer256" bash tools/ab_quick.sh
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
  timeout 400 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "${TESTK:-tma_kernels_match or spitzer or be_pcg or op_apply or virtual or dt_euler or face_kappa or iso}" > gpurun_out/abt_$v.log 2>&1
  echo "$v tests: $(tail -1 gpurun_out/abt_$v.log)"
done
for cfg in ${CFGS:-c3_spitzer256}; do
  for v in $names; do
    if [ $v = prod ]; then unset STS_LIB; else export STS_LIB=$PWD/paper_1610_01265_b200/libsts_b200_$v.so; fi
    timeout 300 python bench.py --config $cfg --steps ${STEPS:-5} --warmup 3 --e2e-steps 0 --no-cpu-baseline ${BARGS:-} > gpurun_out/ab_${cfg}_$v${SUF:-}.log 2>&1
  done
done
unset STS_LIB
if [ -n "$KERNELS" ]; then STS_PCG_HOST_LOOP=1 KERNELS="$KERNELS" bash tools/prof_kernels.sh; fi

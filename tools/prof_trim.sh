mkdir -p gpurun_out
export STS_PCG_HOST_LOOP=1
python tools/profile_step.py --config c4_scale512 --visc > gpurun_out/pp.log 2>&1 || exit 1
K="sts::iso_tma_kernel<.int.6"
for v in prod trim2; do
  if [ $v = prod ]; then unset STS_LIB; else export STS_LIB=$PWD/paper_1610_01265_b200/libsts_b200_$v.so; fi
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$K" -s 3 -c 2 -o gpurun_out/trimprof_$v python tools/profile_step.py --config c4_scale512 --visc > gpurun_out/ncu_trim_$v.log 2>&1
  tail -2 gpurun_out/ncu_trim_$v.log
done
ls gpurun_out

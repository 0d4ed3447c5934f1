# ncu --set full captures of the four hot kernels on the FULL c4 grid (512 x 512 x 1024,
# the bench workload), one launch each; run only after the same command exited 0.
#   bash tools/prof_c4.sh && python tools/make_traffic.py --cells 268435456 gpurun_out/c4prof_*.ncu-rep
mkdir -p gpurun_out
export STS_PCG_HOST_LOOP=1   # (ncu skips kernel nodes of conditional graphs)
rm -f gpurun_out/c4prof_*.ncu-rep
python tools/profile_step.py --config c4_scale512 --visc > gpurun_out/pp.log 2>&1 || exit 1
for K in "sts::aniso_tma_kernel<.int.6" "sts::iso_tma_kernel<.int.6" "sts::aniso_tma_kernel<.int.7" "sts::iso_tma_kernel<.int.7"; do
  tag=$(echo "$K" | tr -c 'a-zA-Z0-9_\n' '_')
  # two consecutive launches: the merged PCG passes alternate a skipped and a catch-up x update
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$K" -s 3 -c 2 -o gpurun_out/c4prof_$tag python tools/profile_step.py --config c4_scale512 --visc > gpurun_out/ncu_$tag.log 2>&1
done
ls gpurun_out

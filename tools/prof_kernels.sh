# ncu captures of the hot kernels (one GPU; run only after the same command exited 0)
# KERNELS: space-separated regexes over demangled names, e.g. "aniso_tma_kernel<.int.2>"
set -x
mkdir -p gpurun_out
CMD="python tools/profile_step.py --config c3_spitzer256 --visc"
$CMD > gpurun_out/plain_prof.log 2>&1 || exit 1
KLIST=${KERNELS:-"aniso_tma_kernel<.int.7,..bool.0,..bool.0> aniso_tma_kernel<.int.6,..bool.0, iso_tma_kernel<.int.7,..int.3,..bool.0,..bool.0> iso_tma_kernel<.int.6,..int.3,..bool.0,"}
for k in $KLIST; do
  tag=$(echo "$k" | tr -c 'a-zA-Z0-9_\n' '_')
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$k" -s 2 -c 1 \
      -o gpurun_out/prof_$tag $CMD > gpurun_out/ncu_$tag.log 2>&1
done
ls -la gpurun_out

# ncu captures of the hot kernels (one GPU; run only after the same command exited 0)
set -x
mkdir -p gpurun_out
python tools/profile_step.py --config c3_spitzer256 --visc > gpurun_out/plain_prof.log 2>&1 || exit 1
for k in ${KERNELS:-"_ZN3sts17aniso_fast_kernelILi2E" "_ZN3sts17aniso_fast_kernelILi4E" "_ZN3sts15iso_fast_kernelILi2ELi3E" "_ZN3sts15iso_fast_kernelILi4ELi3E"}; do
  ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:$k -s 2 -c 1 \
      -o gpurun_out/prof_$k python tools/profile_step.py --config c3_spitzer256 --visc > gpurun_out/ncu_$k.log 2>&1
done
ls -la gpurun_out

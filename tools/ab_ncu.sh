# DRAM bytes / duration of the merged PCG passes for two library variants (c4 grid),
# ncu with a few metrics (one launch each).  VARIANTS: "name=path.so ..." (path "" = product)
set -x
mkdir -p gpurun_out
export STS_PCG_HOST_LOOP=1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second
for pair in $VARIANTS; do
  name=${pair%%=*}; path=${pair#*=}
  if [ -n "$path" ]; then export STS_LIB=$PWD/$path; else unset STS_LIB; fi
  for K in "sts::aniso_tma_kernel<.int.6" "sts::iso_tma_kernel<.int.6" "sts::aniso_tma_kernel<.int.7" "sts::iso_tma_kernel<.int.7"; do
    tag=$(echo "$K" | tr -c 'a-zA-Z0-9_\n' '_')
    ncu --metrics $M --clock-control none --kernel-name-base demangled -k "regex:$K" -s 3 -c 2 --csv \
        python tools/profile_step.py --config c4_scale512 --visc > gpurun_out/abncu_${name}_$tag.csv 2>/dev/null
  done
done

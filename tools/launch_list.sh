# per-launch device times of our kernels for one bench step (cold-cache, serialised)
set -x
mkdir -p gpurun_out
# (ncu skips the kernel nodes of graphs with conditional nodes: the PCG kernels are
#  launched from the host-polled loop for this capture, STS_PCG_HOST_LOOP=1)
export STS_PCG_HOST_LOOP=1
CMD="python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline"
$CMD > gpurun_out/bench_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:sts:: -c 6000 \
    --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
tail -3 gpurun_out/ncu_launches.log

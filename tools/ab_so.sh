# A-B of prebuilt library files on the default bench (same box, interleaved runs).
#   SOS="old=paper_1610_01265_b200/libsts_b200_old.so new=" bash tools/ab_so.sh   (empty path = product)
set -x
mkdir -p gpurun_out
for round in 1 2; do
  for pair in $SOS; do
    v=${pair%%=*}; path=${pair#*=}
    if [ -n "$path" ]; then export STS_LIB=$PWD/$path; else unset STS_LIB; fi
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

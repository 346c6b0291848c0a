#!/bin/bash
# Same-box comparison of several builds of the library, alternating, twice each:
#   scripts/abn.sh TAG "LIB1 LIB2 ..." "WORKLOAD STEPS" ["WORKLOAD STEPS" ...]
# LIBn are library paths (PGPCV_LIB); bench lines land in
# gpurun_out/bench_TAG_<workload>_<n>_<rep>.json (n = position in the list).
set -u
tag=$1; libs=($2); shift 2
jobs=("$@")
mkdir -p gpurun_out
for rep in 1 2; do
  for w in "${jobs[@]}"; do
    read -r wl steps <<< "$w"
    n=0
    for lib in "${libs[@]}"; do
      PGPCV_LIB=$lib bash scripts/gpu_job.sh bench ${tag}_${wl}_${n}_$rep --workload $wl --steps $steps --no-cpu-baseline
      n=$((n+1))
    done
  done
done
for f in gpurun_out/bench_${tag}_*.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value'],1), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])"; done

#!/bin/bash
# Same-box A/B of two builds or settings of the library, alternating, twice each:
#   scripts/ab.sh TAG "ENV_A" "ENV_B" "WORKLOAD STEPS" ["WORKLOAD STEPS" ...]
# ENV_A / ENV_B are environment assignments for bench.py, e.g.
#   "PGPCV_LIB=paper_1912_13132_b200/libpgpcv_ps0.so" (a variant build: _build.build(defines=..., out=...))
#   "PGPCV_SIGMA_REUSE=0" / "PGPCV_WS=1" / "X=1" (a no-op for the default build)
# Bench lines land in gpurun_out/bench_TAG_<workload>_{a,b}_<rep>.json (run from the repo root,
# through gpurun; the round-2 A/B records under profiles/r02_ab_*.json came from this pattern).
set -u
tag=$1; envA=$2; envB=$3; shift 3
jobs=("$@")
mkdir -p gpurun_out
for rep in 1 2; do
  for w in "${jobs[@]}"; do
    read -r wl steps <<< "$w"
    env $envA bash scripts/gpu_job.sh bench ${tag}_${wl}_a_$rep --workload $wl --steps $steps --no-cpu-baseline
    env $envB bash scripts/gpu_job.sh bench ${tag}_${wl}_b_$rep --workload $wl --steps $steps --no-cpu-baseline
  done
done

#!/bin/bash
# The round's judged measurements on one box: the GPU suite + smoke, the headline bench line
# (c5, default), the other workloads and modes, the reference arm, then the ncu launch list of
# the default bench and one full capture of a c5 cv_kernel launch.  `grid` as second argument
# adds the whole-grid call (10 min).
set -u
mkdir -p gpurun_out
tag=${1:-final}
bash scripts/gpu_job.sh tests
bash scripts/gpu_job.sh bench ${tag}_c5
[ "${2:-}" = grid ] && bash scripts/gpu_job.sh bench ${tag}_c5_grid125 --configs-per-step 125 --steps 2 --warmup 3 --no-cpu-baseline
for m in cv_nll nll predict gls; do bash scripts/gpu_job.sh bench ${tag}_c5_$m --mode $m --steps 3 --no-cpu-baseline; done
bash scripts/gpu_job.sh bench ${tag}_c6 --workload c6 --steps 2 --no-cpu-baseline
bash scripts/gpu_job.sh bench ${tag}_c4 --workload c4 --steps 15 --no-cpu-baseline
bash scripts/gpu_job.sh bench ${tag}_c3 --workload c3 --steps 150 --no-cpu-baseline
bash scripts/gpu_job.sh bench ${tag}_c2 --workload c2 --steps 400 --no-cpu-baseline
bash scripts/gpu_job.sh bench ${tag}_reference --impl reference --steps 2 --warmup 3
bash scripts/gpu_job.sh launches ${tag} --steps 2 --warmup 1
bash scripts/gpu_job.sh ncufull ${tag}_c5

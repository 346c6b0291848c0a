#!/bin/bash
# GPU-box jobs (run through gpurun from the repo root): outputs land in gpurun_out/.
#   scripts/gpu_job.sh tests            -m gpu suite + smoke
#   scripts/gpu_job.sh bench TAG [args] bench.py line -> gpurun_out/bench_TAG.json
#   scripts/gpu_job.sh parity PLAN      scripts/parity_report.py --plan PLAN
#   scripts/gpu_job.sh launches TAG     ncu launch list of the default bench
#   scripts/gpu_job.sh ncufull TAG [args] ncu --set full capture of one cv_kernel launch
set -u
mkdir -p gpurun_out
job=$1; shift
case "$job" in
  tests)
    nproc > gpurun_out/nproc.txt
    timeout 2400 python -m pytest tests -m gpu -q -rA --durations=15 > gpurun_out/pytest_gpu.log 2>&1
    echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
    timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
    echo "smoke rc $?" >> gpurun_out/smoke.log ;;
  bench)
    tag=$1; shift
    timeout 1800 python bench.py "$@" > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
    echo "bench $tag rc $?" >> gpurun_out/bench_$tag.err ;;
  parity)
    timeout 5400 python scripts/parity_report.py --plan "$1" > gpurun_out/parity_$1.json 2> gpurun_out/parity_$1.err
    echo "parity rc $?" >> gpurun_out/parity_$1.err ;;
  launches)
    tag=$1; shift
    timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches_$tag.csv python bench.py --no-cpu-baseline "$@" > gpurun_out/ncu_launch_$tag.log 2>&1 ;;
  ncufull)
    tag=$1; shift
    timeout 2400 ncu --set full --import-source on --clock-control none -k regex:cv_kernel -c 1 \
      -o gpurun_out/prof_$tag python bench.py --steps 1 --warmup 0 --configs-per-step 1 --no-cpu-baseline "$@" \
      > gpurun_out/ncu_full_$tag.log 2>&1 ;;
  phases)
    timeout 900 python probes/p2_phases.py "$1" > gpurun_out/p2_$1_${2:-default}.json 2> gpurun_out/p2_$1_${2:-default}.err ;;
  *) echo "unknown job $job"; exit 2 ;;
esac

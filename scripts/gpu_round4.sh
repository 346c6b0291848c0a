# GPU: two-ended scheduling experiment (PGPCV_SCHED 0 vs 1) + tests
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "two_ended or repeated or c2_full" > gpurun_out/pytest_sched.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_sched.log
for s in 0 1; do
  PGPCV_SCHED=$s timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_c5_s$s.json 2> gpurun_out/bench_c5_s$s.err
  PGPCV_SCHED=$s timeout 600 python probes/p2_phases.py c5 > gpurun_out/p2_c5_s$s.json 2>&1
done
for s in 0 1; do
  PGPCV_SCHED=$s timeout 900 python bench.py --workload c6 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_c6_s$s.json 2> gpurun_out/bench_c6_s$s.err
done
echo done

# A/B jobs of round 2 (second session): per-range covariance reuse (small kernel), the
# consumer-side loop fence (large and small kernels), P6 KC = 8 operand-ring variants.
set -u
mkdir -p gpurun_out
NF=paper_1912_13132_b200/libpgpcv_nofence.so
timeout 900 python -m pytest tests/test_gpu_sigma.py -x -q -rA > gpurun_out/pytest_sigma.log 2>&1; echo "rc $?" >> gpurun_out/pytest_sigma.log
timeout 600 ./probes/p6_protocol -1 2 > gpurun_out/p6_kc8.json 2> gpurun_out/p6_kc8.err
for rep in 1 2; do
  for w in "c3 150" "c2 400" "c4 15"; do
    set -- $w
    PGPCV_SIGMA_REUSE=0 bash scripts/gpu_job.sh bench ${1}_off_$rep --workload $1 --steps $2 --no-cpu-baseline
    bash scripts/gpu_job.sh bench ${1}_on_$rep --workload $1 --steps $2 --no-cpu-baseline
  done
done
(PGPCV_LIB=$NF timeout 900 python probes/stress_c2.py 20 > gpurun_out/stress_nofence_small.log 2>&1;
 PGPCV_LIB=$NF PGPCV_SMALL_K=0 timeout 900 python probes/stress_c2.py 20 > gpurun_out/stress_nofence_large.log 2>&1)
for rep in 1 2; do
  bash scripts/gpu_job.sh bench c5_fence_$rep --steps 3 --no-cpu-baseline
  PGPCV_LIB=$NF bash scripts/gpu_job.sh bench c5_nofence_$rep --steps 3 --no-cpu-baseline
done
PGPCV_LIB=$NF timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_nofence.log 2>&1; echo "rc $?" >> gpurun_out/pytest_nofence.log

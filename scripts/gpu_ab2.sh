# A/B on one box: previous kernel (probes/libpgpcv_prev.so) vs the tree's (branch-free sqrt); + tests
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
for r in 1 2; do
  PGPCV_LIB=$PWD/probes/libpgpcv_prev.so timeout 900 python bench.py --no-cpu-baseline --steps 3 --warmup 2 > gpurun_out/ab_prev_$r.json 2>/dev/null
  timeout 900 python bench.py --no-cpu-baseline --steps 3 --warmup 2 > gpurun_out/ab_new_$r.json 2>/dev/null
done
for w in c3 c4; do
  PGPCV_LIB=$PWD/probes/libpgpcv_prev.so timeout 900 python bench.py --workload $w --no-cpu-baseline > gpurun_out/ab_prev_$w.json 2>/dev/null
  timeout 900 python bench.py --workload $w --no-cpu-baseline > gpurun_out/ab_new_$w.json 2>/dev/null
done
timeout 600 python probes/p2_phases.py c5 > gpurun_out/p2_c5.json 2>&1
echo done

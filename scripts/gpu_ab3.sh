# Same-box A/B: probes/libpgpcv_prev.so vs the tree's lib on c3/c4 (x2, interleaved) and c5; + GPU tests + c3 phases
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
for r in 1 2; do
  for w in c3 c4; do
    PGPCV_LIB=$PWD/probes/libpgpcv_prev.so timeout 900 python bench.py --workload $w --no-cpu-baseline > gpurun_out/ab_prev_${w}_$r.json 2>/dev/null
    timeout 900 python bench.py --workload $w --no-cpu-baseline > gpurun_out/ab_new_${w}_$r.json 2>/dev/null
  done
done
PGPCV_LIB=$PWD/probes/libpgpcv_prev.so timeout 900 python bench.py --no-cpu-baseline --steps 3 --warmup 2 > gpurun_out/ab_prev_c5.json 2>/dev/null
timeout 900 python bench.py --no-cpu-baseline --steps 3 --warmup 2 > gpurun_out/ab_new_c5.json 2>/dev/null
timeout 600 python probes/p2_phases.py c3 > gpurun_out/p2_c3.json 2>&1
echo done

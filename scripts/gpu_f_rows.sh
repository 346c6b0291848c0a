# GPU: GLS parity (row f4) and measurements of the NEXT rows (f1 predict, f2 c6, f3 nll).
set -x
timeout 1200 python -m pytest tests/test_gpu_gls.py -x -q -rA --durations=0 > gpurun_out/pytest_gls.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gls.log
for m in cv_nll nll predict; do
  timeout 600 python bench.py --mode $m --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5_$m.json 2> gpurun_out/bench_c5_$m.err
done
timeout 900 python bench.py --workload c6 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c6_cv.json 2> gpurun_out/bench_c6_cv.err
echo done

set -x
timeout 1500 python -m pytest tests -m gpu -x -q -rA --durations=8 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
for w in c2 c3 c4; do timeout 900 python bench.py --workload $w --no-cpu-baseline > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; done
for sk in 256 384 640; do PGPCV_SMALL_K=$sk timeout 900 python bench.py --workload c4 --no-cpu-baseline > gpurun_out/bench_c4_sk$sk.json 2> gpurun_out/bench_c4_sk$sk.err; done
timeout 900 python bench.py --no-cpu-baseline --steps 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
echo done

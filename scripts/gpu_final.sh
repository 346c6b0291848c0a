# GPU: final verification of the round's tree -- -m gpu suite, smoke, default bench, launch list, ncu full
set -x
nproc > gpurun_out/nproc.txt
timeout 1500 python -m pytest tests -m gpu -q -rA --durations=10 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 python bench.py --workload c6 --configs-per-step 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c6_cv.json 2> gpurun_out/bench_c6_cv.err
for w in c3 c4; do timeout 900 python bench.py --workload $w --no-cpu-baseline > gpurun_out/bench_$w.json 2>/dev/null; done
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py > gpurun_out/ncu_launch.log 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:cv_kernel -c 1 -o gpurun_out/prof_cv_v12 python bench.py --steps 1 --warmup 0 --configs-per-step 1 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
echo done

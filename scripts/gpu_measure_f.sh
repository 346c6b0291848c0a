# GPU: rows f1-f4 measured on the final kernel (c5), plus the default bench line with partition time
set -x
timeout 900 python bench.py > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
for m in cv_nll nll predict gls; do
  timeout 900 python bench.py --mode $m --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5_$m.json 2> gpurun_out/bench_c5_$m.err
done
echo done

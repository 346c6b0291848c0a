# Rows f1-f4 on the tree's kernel: c5 in every evaluation mode (one bench line each)
set -x
for m in cv_nll nll predict gls; do
  timeout 900 python bench.py --mode $m --no-cpu-baseline > gpurun_out/bench_c5_$m.json 2> gpurun_out/bench_c5_$m.err
done
echo done

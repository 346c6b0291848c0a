# GPU: L2 prefetch distance A/B (PFD 2/4/8) on c5; c2/c3/c4 throughput
set -x
for v in pfd2 pfd8; do
  PGPCV_LIB=$PWD/probes/libpgpcv_$v.so timeout 900 python bench.py --no-cpu-baseline --steps 3 > gpurun_out/bench_c5_$v.json 2> gpurun_out/bench_c5_$v.err
done
timeout 900 python bench.py --no-cpu-baseline --steps 3 > gpurun_out/bench_c5_pfd4.json 2> gpurun_out/bench_c5_pfd4.err
for w in c2 c3 c4; do
  timeout 900 python bench.py --workload $w --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
done
echo done

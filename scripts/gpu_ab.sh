# A/B on one box: previous kernel (probes/libpgpcv_v9.so) vs the tree's kernel, alternating
set -x
for r in 1 2; do
  PGPCV_LIB=$PWD/probes/libpgpcv_v9.so timeout 900 python bench.py --no-cpu-baseline --steps 3 --warmup 2 > gpurun_out/ab_v9_$r.json 2>/dev/null
  timeout 900 python bench.py --no-cpu-baseline --steps 3 --warmup 2 > gpurun_out/ab_new_$r.json 2>/dev/null
done
echo done

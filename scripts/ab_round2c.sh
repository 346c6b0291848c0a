# Same-box A/B: HEAD-of-session library vs the per-range reuse build (reuse off / on) and the
# no-loop-fence build; P2 phases of the small kernel at c3 with the reuse.
set -u
mkdir -p gpurun_out
H=paper_1912_13132_b200/libpgpcv_head.so
NF=paper_1912_13132_b200/libpgpcv_nofence.so
for rep in 1 2; do
  for w in "c3 150" "c4 15"; do
    set -- $w
    PGPCV_LIB=$H bash scripts/gpu_job.sh bench ${1}_head_$rep --workload $1 --steps $2 --no-cpu-baseline
    PGPCV_SIGMA_REUSE=0 bash scripts/gpu_job.sh bench ${1}_off_$rep --workload $1 --steps $2 --no-cpu-baseline
    bash scripts/gpu_job.sh bench ${1}_on_$rep --workload $1 --steps $2 --no-cpu-baseline
    PGPCV_LIB=$NF bash scripts/gpu_job.sh bench ${1}_nf_$rep --workload $1 --steps $2 --no-cpu-baseline
  done
done
P2_STEP=1 timeout 900 python probes/p2_phases.py c3 > gpurun_out/p2_c3_step_reuse.json 2> gpurun_out/p2_c3_step_reuse.err
P2_STEP=1 PGPCV_SIGMA_REUSE=0 timeout 900 python probes/p2_phases.py c3 > gpurun_out/p2_c3_step_noreuse.json 2> gpurun_out/p2_c3_step_noreuse.err

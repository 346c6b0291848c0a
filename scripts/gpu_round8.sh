set -x
for w in c2 c3 c4; do timeout 600 python probes/p2_phases.py $w > gpurun_out/p2_$w.json 2>&1; done
echo done

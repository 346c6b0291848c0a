set -x
for w in c3 c5; do timeout 600 python probes/p2_phases.py $w > gpurun_out/p2_$w.json 2>&1; done
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke.log
echo done

set -x
timeout 900 python probes/p3_timeline.py c5 > gpurun_out/p3_c5.json 2>&1
echo done

# GPU check of the current tree: the -m gpu suite, the DMMA inner-loop probe.
set -x
./probes/p1_dmma_loop > gpurun_out/p1.json 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -rA > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
echo done

set -x
timeout 1500 python -m pytest tests/test_gpu_bisect.py -x -q -rA --durations=0 > gpurun_out/pytest_bisect.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_bisect.log
echo done

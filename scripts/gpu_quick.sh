set -x
timeout 1200 python -m pytest tests/test_gpu_edge.py -x -q > gpurun_out/pytest_edge.log 2>&1; echo "pytest rc=$?"; tail -25 gpurun_out/pytest_edge.log

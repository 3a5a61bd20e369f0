set -x
timeout 1200 python -m pytest tests/test_gpu_distributed.py -x -q > gpurun_out/pytest_gpu_dist.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu_dist.log

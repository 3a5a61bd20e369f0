timeout 900 python -m pytest tests/test_gpu_distributed.py tests/test_gpu_index.py -x -q > gpurun_out/pytest_d.log 2>&1; echo "rc=$?"; tail -15 gpurun_out/pytest_d.log

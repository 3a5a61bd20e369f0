set -x
timeout 2400 python -m pytest tests/test_gpu_parity.py -x -q -k large_sampled --durations=5 > gpurun_out/pytest_large.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_large.log

timeout 900 python -m pytest tests/test_gpu_index.py -x -q > gpurun_out/pytest_idx.log 2>&1; echo "idx rc=$?"; tail -15 gpurun_out/pytest_idx.log
timeout 900 python scripts/configs_probe.py c1 ncc+index 6 > gpurun_out/p_idx.log 2>&1; echo "rc=$?"; cat gpurun_out/p_idx.log | cut -c1-420

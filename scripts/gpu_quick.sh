timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -25 gpurun_out/pytest_gpu.log
SSKM_DEBUG=1 timeout 600 python scripts/configs_probe.py c0 ncc 8 > gpurun_out/p_c0.log 2>&1; echo "c0 rc=$?"; grep -E "iter" gpurun_out/p_c0.log | tail -3 | cut -c1-200
SSKM_DEBUG=1 timeout 900 python scripts/configs_probe.py c2 baseline 3 > gpurun_out/p_c2.log 2>&1; echo "c2 rc=$?"; grep -E "sskm|iter" gpurun_out/p_c2.log | tail -4 | cut -c1-200

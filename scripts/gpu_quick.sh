set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "approximate or teacher_forced_c0" > gpurun_out/pytest_eps.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_eps.log
timeout 900 python scripts/configs_probe.py c2 ncc 14 > gpurun_out/c2ncc.log 2>&1; echo "c2 rc=$?"; grep iter gpurun_out/c2ncc.log | cut -c1-260

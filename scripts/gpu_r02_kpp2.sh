timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bound.py tests/test_gpu_multi.py -x -q > gpurun_out/pytest_kpp2.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_kpp2.log
timeout 600 python scripts/probe_kpp.py c1
timeout 900 python scripts/probe_kpp.py c2
source scripts/_run_probe.sh
run wg c1 34

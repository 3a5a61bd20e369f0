timeout 900 python -m pytest tests/test_gpu_bound.py tests/test_gpu_parity.py tests/test_gpu_multi.py -x -q > gpurun_out/pytest_maint.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_maint.log
source scripts/_run_probe.sh
run maint c1 34
run maint c0 20




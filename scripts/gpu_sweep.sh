set -x
timeout 600 python scripts/assign_sweep.py c1 > gpurun_out/sweep_c1.log 2>&1; echo "sweep rc=$?"
cat gpurun_out/sweep_c1.log | tail -20
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log

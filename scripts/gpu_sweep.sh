set -x
timeout 900 python scripts/assign_sweep.py c1 > gpurun_out/sweep_c1.log 2>&1; echo "sweep rc=$?"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log

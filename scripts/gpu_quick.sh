set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
timeout 600 python scripts/density_probe.py c1 > gpurun_out/probe_c1.log 2>&1; echo "probe rc=$?"; cat gpurun_out/probe_c1.log | grep "^{"

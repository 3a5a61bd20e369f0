set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python scripts/configs_probe.py c1 baseline 5 > gpurun_out/p.log 2>&1; echo "c1 rc=$?"; tail -1 gpurun_out/p.log | cut -c1-120
CMD="python scripts/configs_probe.py c1 baseline 2"
$CMD > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_probe.csv $CMD > gpurun_out/ncu_l.log 2>&1; echo "ncu rc=$?"

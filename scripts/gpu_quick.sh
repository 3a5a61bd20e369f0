set -x
for c in c1 c4; do timeout 900 python scripts/configs_probe.py $c baseline 3 > gpurun_out/p_$c.log 2>&1; echo "$c rc=$?"; tail -1 gpurun_out/p_$c.log | cut -c1-120; done
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log

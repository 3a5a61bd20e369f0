set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for c in c3 c1; do
  timeout 900 python scripts/configs_probe.py $c ncc 8 > gpurun_out/cfg_$c.log 2>&1; echo "$c rc=$?"; grep "^{" gpurun_out/cfg_$c.log | tail -4
done

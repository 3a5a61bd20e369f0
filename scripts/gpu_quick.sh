set -x
for lib in paper_2108_00895_b200/libsskm_b200.so paper_2108_00895_b200/libsskm_b200_l1.so; do
  SSKM_LIB=$PWD/$lib timeout 600 python scripts/configs_probe.py c1 baseline 5 > gpurun_out/p.log 2>&1; echo "$lib rc=$?"; tail -1 gpurun_out/p.log | cut -c1-120
  SSKM_LIB=$PWD/$lib timeout 600 python scripts/configs_probe.py c4 baseline 1 > gpurun_out/p4.log 2>&1; echo "$lib c4 rc=$?"; tail -1 gpurun_out/p4.log | cut -c1-120
done
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log

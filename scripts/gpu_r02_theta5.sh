source scripts/_run_probe.sh
run default c1 34
run default c3 14
run default c0 20
run default c2 10
run default c4 8
timeout 1200 python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_parity_large.py > gpurun_out/pytest_t5.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_t5.log

# round 2: new large parity tests + the rest of the GPU suite + bench
free -g | head -2; nproc
timeout 2400 python -m pytest tests/test_gpu_parity_large.py -x -q -s --durations=0 > gpurun_out/pytest_large.log 2>&1; echo "large rc=$?"; tail -15 gpurun_out/pytest_large.log
timeout 1500 python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_parity_large.py > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log | cut -c1-3000

nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 2400 python -m pytest tests -m gpu -x -q --durations=10 > gpurun_out/s4_pytest.log 2>&1; echo "pytest rc=$?"; tail -16 gpurun_out/s4_pytest.log
timeout 300 python __graft_entry__.py > gpurun_out/s4_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/s4_smoke.log
timeout 900 python bench.py > gpurun_out/s4_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/s4_bench.log | cut -c1-1500
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/s4_bench_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/s4_bench_ref.log | cut -c1-800

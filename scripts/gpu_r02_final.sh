nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 2400 python -m pytest tests -m gpu -x -q --durations=6 > gpurun_out/final_pytest.log 2>&1; echo "pytest rc=$?"; tail -12 gpurun_out/final_pytest.log
timeout 300 python __graft_entry__.py > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/final_smoke.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/final_bench_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/final_bench_ref.log | cut -c1-400
timeout 900 python bench.py > gpurun_out/final_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/final_bench.log | cut -c1-1300
timeout 900 python bench.py --mode ncc --no-e2e --no-cpu-baseline > gpurun_out/final_bench_ncc.log 2>&1; echo "ncc rc=$?"; tail -1 gpurun_out/final_bench_ncc.log | cut -c1-300

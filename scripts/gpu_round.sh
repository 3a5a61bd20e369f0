# one GPU pass: smoke, GPU parity suite, short bench, ncu launch list of the bench command
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
CMD="python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline"
SSKM_DEBUG=1 timeout 600 $CMD > gpurun_out/plain.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/plain.log | cut -c1-600; grep sskm gpurun_out/plain.log | tail -4
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
echo "launches rc=$?"

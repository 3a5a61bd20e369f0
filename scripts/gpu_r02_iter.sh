# round 2 iteration: GPU suite (incl. large parity) + bench + launch list + bound-screen ncu capture
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log | cut -c1-4000
CMD="python bench.py --steps 3 --warmup 20 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bound_screen_kernel" -s 21 -c 1 -o gpurun_out/prof_bound $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu bound rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"write_groups|hipost_build|delta_local" -s 63 -c 3 -o gpurun_out/prof_upd $CMD > gpurun_out/ncu_upd.log 2>&1; echo "ncu upd rc=$?"

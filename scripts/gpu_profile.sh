# ncu evidence for the assign kernel (run under gpurun; 1 GPU)
set -x
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
echo "launches rc=$?"
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:assign_kernel -s 3 -c 1 -o gpurun_out/prof_assign $CMD > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
$CMD > gpurun_out/plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"write_cols|delta_local|norm2" -s 0 -c 3 -o gpurun_out/prof_update $CMD > gpurun_out/ncu_full_upd.log 2>&1
echo "full-update rc=$?"
ls -la gpurun_out

P="python scripts/probe_drift.py c1 30 --stats-only"
$P > gpurun_out/s4f_probe_plain.log 2>&1; echo "plain rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bound_screen_kernel" -s 27 -c 1 -o gpurun_out/s4f_prof_bound $P > gpurun_out/s4f_probe_bound.log 2>&1; echo "ncu bound rc=$?"; grep '"it": 28' gpurun_out/s4f_probe_bound.log | cut -c1-700
timeout 900 ncu --set full --clock-control none -k regex:"bound_screen_kernel" -s 7 -c 1 -o gpurun_out/s4f_prof_bound8 $P > gpurun_out/s4f_probe_bound8.log 2>&1; echo "ncu bound8 rc=$?"; grep '"it": 8,' gpurun_out/s4f_probe_bound8.log | cut -c1-700
CMD="python bench.py --steps 3 --warmup 27 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/s4f_plain_prof.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s4f_launches_steady.csv $CMD > gpurun_out/s4f_ncu_launches.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none -k regex:"write_groups|hipost_build|skip_kernel|delta_local|group_drift" -s 40 -c 8 -o gpurun_out/s4f_prof_upd $P > gpurun_out/s4f_probe_upd.log 2>&1; echo "ncu upd rc=$?"

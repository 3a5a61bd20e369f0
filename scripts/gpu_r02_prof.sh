# round-2 evidence: e2e phases, steady-state launch list, full ncu captures (bound screen, update kernels)
SSKM_DEBUG=1 python scripts/e2e_phases.py > gpurun_out/e2e_phases.log 2>&1; echo "e2e rc=$?"; grep -v "bound init" gpurun_out/e2e_phases.log | tail -12
CMD="python bench.py --steps 3 --warmup 27 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_prof.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_steady.csv $CMD > gpurun_out/ncu_launches.log 2>&1; echo "launches rc=$?"
P="python scripts/probe_drift.py c1 30 --stats-only"
$P > gpurun_out/probe_prof_plain.log 2>&1; echo "plain rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bound_screen_kernel" -s 27 -c 1 -o gpurun_out/r02_prof_bound $P > gpurun_out/probe_prof_bound.log 2>&1; echo "ncu bound rc=$?"; grep '"it": 28' gpurun_out/probe_prof_bound.log | cut -c1-600
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"write_groups|hipost_build|skip_kernel|delta_local|reduce_groups" -s 100 -c 6 -o gpurun_out/r02_prof_upd $P > gpurun_out/probe_prof_upd.log 2>&1; echo "ncu upd rc=$?"

# source-level ncu of the bound screen at an early (all documents screened) and a late iteration; update kernels
P="python scripts/probe_drift.py c1 30 --stats-only"
$P > gpurun_out/s4_probe_plain.log 2>&1; echo "plain rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bound_screen_kernel" -s 7 -c 1 -o gpurun_out/s4_prof_bound_it8 $P > gpurun_out/s4_probe_b8.log 2>&1; echo "ncu bound8 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bound_screen_kernel" -s 27 -c 1 -o gpurun_out/s4_prof_bound_it28 $P > gpurun_out/s4_probe_b28.log 2>&1; echo "ncu bound28 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"write_groups|hipost_build|skip_kernel|delta_local|reduce_groups|moved_kernel|flags_kernel" -s 70 -c 10 -o gpurun_out/s4_prof_upd $P > gpurun_out/s4_probe_upd.log 2>&1; echo "ncu upd rc=$?"

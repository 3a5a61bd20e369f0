# bound screen source-level profile at a steady iteration (c1 baseline) + update kernels
P="python scripts/probe_drift.py c1 24 --stats-only"
$P > gpurun_out/src_plain.log 2>&1; echo "plain rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bound_screen_kernel" -s 20 -c 1 -o gpurun_out/r02_src_bound $P > gpurun_out/src_ncu.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/r02_src_bound.ncu-rep --page source --csv --print-source sass > gpurun_out/r02_src_bound_sass.csv 2>&1; echo "sass rc=$?"
ncu -i gpurun_out/r02_src_bound.ncu-rep --page source --csv --print-source cuda > gpurun_out/r02_src_bound_cuda.csv 2>&1; echo "cuda rc=$?"
ncu -i gpurun_out/r02_src_bound.ncu-rep --page raw --csv > gpurun_out/r02_src_bound_raw.csv 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"write_groups|hipost|skip_kernel|delta_local|reduce_groups|moved_kernel|flags_kernel" -s 60 -c 8 -o gpurun_out/r02_src_upd $P > gpurun_out/src_ncu_upd.log 2>&1; echo "ncu upd rc=$?"
ncu -i gpurun_out/r02_src_upd.ncu-rep --page raw --csv > gpurun_out/r02_src_upd_raw.csv 2>&1
ls -la gpurun_out

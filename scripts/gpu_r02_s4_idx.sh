python scripts/configs_probe.py c1 ncc 8 > gpurun_out/s4_c1_ncc.log 2>&1; echo "ncc rc=$?"; tail -3 gpurun_out/s4_c1_ncc.log | cut -c1-400
python scripts/configs_probe.py c1 ncc+index 8 > gpurun_out/s4_c1_nccidx.log 2>&1; echo "nccidx rc=$?"; tail -3 gpurun_out/s4_c1_nccidx.log | cut -c1-500
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s4_idx_launches.csv python scripts/configs_probe.py c1 ncc+index 6 > gpurun_out/s4_idx_ncu.log 2>&1; echo "launches rc=$?"

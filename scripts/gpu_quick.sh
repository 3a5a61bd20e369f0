for R in 0 1; do
  SSKM_RECORD_OWN=$R timeout 600 python scripts/configs_probe.py c1 baseline 5 > gpurun_out/p_$R.log 2>&1; echo "R=$R rc=$?"; tail -3 gpurun_out/p_$R.log | cut -c1-130
done
timeout 300 python scripts/prof_one.py c1 3 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum --clock-control none -k regex:"^resolve_kernel|^postings_screen" -s 2 -c 4 python scripts/prof_one.py c1 3 > gpurun_out/ncu_res.log 2>&1
echo "ncu rc=$?"; grep -E "resolve_kernel|postings_screen|duration|inst_exec|dram" gpurun_out/ncu_res.log | cut -c1-80 | head -16

# ncu full captures of the bound screen and its init (1 GPU)
set -x
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/plain.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/plain.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], json.dumps(d['roofline'])[:900], d['phase_ms'])"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bound_screen_kernel" -s 3 -c 1 -o gpurun_out/prof_bound $CMD > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bound_init_kernel" -s 3 -c 1 -o gpurun_out/prof_binit $CMD > gpurun_out/ncu_full2.log 2>&1; echo "full2 rc=$?"

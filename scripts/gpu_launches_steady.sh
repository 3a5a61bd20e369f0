set -x
CMD="python bench.py --steps 2 --warmup 24 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_steady.csv $CMD > gpurun_out/ncu_ls.log 2>&1; echo "rc=$?"

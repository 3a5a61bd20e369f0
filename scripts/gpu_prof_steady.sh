# ncu full capture of the bound screen at steady state (theta converged): c1, 24 warm-up iterations
set -x
CMD="python bench.py --steps 2 --warmup 24 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bound_screen_kernel" -s 24 -c 1 -o gpurun_out/prof_steady $CMD > gpurun_out/ncu_steady.log 2>&1; echo "ncu rc=$?"

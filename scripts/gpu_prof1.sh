# ncu full capture of one kernel of the c1 bench: KPAT=<regex> OUT=<name>
set -x
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KPAT" -s ${SKIP:-3} -c 1 -o gpurun_out/$OUT $CMD > gpurun_out/ncu_$OUT.log 2>&1; echo "ncu rc=$?"

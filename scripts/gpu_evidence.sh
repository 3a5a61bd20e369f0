# round evidence: smoke, full bench line, reference arm, ncu launch list + bound-screen capture (1 GPU)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_full.log | cut -c1-300
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bound_screen_kernel" -s 3 -c 1 -o gpurun_out/prof_bound_final $CMD > gpurun_out/ncu_prof_final.log 2>&1; echo "ncu rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench_ref.log | cut -c1-300
for c in c0 c1 c2 c3; do
timeout 900 python scripts/configs_probe.py $c baseline 12 > gpurun_out/cfg_$c.log 2>&1; echo "$c rc=$?"; tail -1 gpurun_out/cfg_$c.log | cut -c1-250
done

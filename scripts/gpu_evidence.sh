# round evidence: full bench line, reference arm, ncu launch list, per-config probes (1 GPU)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
nproc; lscpu | grep "Model name"
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_full.log | cut -c1-300
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1; echo "launches rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench_ref.log | cut -c1-300
for c in c0 c1 c2 c3; do
timeout 900 python scripts/configs_probe.py $c baseline 8 > gpurun_out/cfg_$c.log 2>&1; echo "$c rc=$?"; tail -1 gpurun_out/cfg_$c.log | cut -c1-250
done
timeout 1500 python scripts/configs_probe.py c4 baseline 4 > gpurun_out/cfg_c4.log 2>&1; echo "c4 rc=$?"; tail -1 gpurun_out/cfg_c4.log | cut -c1-250

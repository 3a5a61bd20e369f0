nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 2400 python -m pytest tests -m gpu -x -q --durations=6 > gpurun_out/s4_pytest3.log 2>&1; echo "pytest rc=$?"; tail -12 gpurun_out/s4_pytest3.log
timeout 300 python __graft_entry__.py > gpurun_out/s4_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/s4_smoke.log
timeout 900 python bench.py > gpurun_out/s4_bench2.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/s4_bench2.log | cut -c1-1800
for c in c2 c4; do
timeout 1200 python bench.py --config $c --steps 12 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s4_bench2_$c.log 2>/dev/null; echo "$c rc=$?"; tail -1 gpurun_out/s4_bench2_$c.log | python -c "
import json,sys; x=json.loads(sys.stdin.read()); print(x['config']['workload'][:40], x['ms_per_step'], x['phase_ms'], x.get('exact_scan_docs_per_iter'), x['drift_bound']['docs_kept_per_iter'], x['clocks'])"
done

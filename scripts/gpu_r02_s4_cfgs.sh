timeout 900 python -m pytest tests/test_gpu_bound.py -x -q > gpurun_out/s4_bound_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s4_bound_pytest.log
for c in c0 c2 c3; do
timeout 1200 python bench.py --config $c --steps 12 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s4_bench_$c.log 2>/dev/null; echo "$c rc=$?"; tail -1 gpurun_out/s4_bench_$c.log | python -c "
import json,sys; x=json.loads(sys.stdin.read()); print(x['config']['workload'][:40], x['ms_per_step'], x['phase_ms'], x.get('exact_scan_docs_per_iter'), x['clocks'], x.get('parity',{}).get('ok'))"
done
P="python scripts/probe_drift.py c1 30 --stats-only"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"write_groups|hipost_build|skip_kernel|delta_local|reduce_groups|moved_kernel|flags_kernel" -s 70 -c 10 -o gpurun_out/s4_prof_upd2 $P > gpurun_out/s4_probe_upd2.log 2>&1; echo "ncu upd rc=$?"

timeout 900 python -m pytest tests/test_gpu_bound.py tests/test_gpu_parity.py tests/test_gpu_multi.py -x -q > gpurun_out/pytest_skip.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_skip.log
python scripts/probe_drift.py c1 30 > gpurun_out/probe_drift4.log 2>&1; echo "probe rc=$?"; python - <<'PY'
import json
for l in open('gpurun_out/probe_drift4.log'):
    if l.startswith('{'):
        d=json.loads(l); print(d['it'], round(d['ms'],3), 'upd', round(d['upd'],3), 'asg', round(d['asg'],3), 'scr', round(d['screen'],3), 'skip', d['skip_docs'], round(d['skip_ms'],3), d['skip_own'], 'moved', d['moved'], 'rec', d['recomputed'])
PY
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_skip3.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_skip3.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['iteration_ms']['warmup'], d['iteration_ms']['last_5_mean'], d['phase_ms'], d['drift_bound'], d['e2e']['value'], d['e2e']['wall_s'])"
CMD="python bench.py --steps 3 --warmup 27 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_skip.csv $CMD > gpurun_out/ncu_launches.log 2>&1; echo "launches rc=$?"

timeout 900 python -m pytest tests/test_gpu_bound.py tests/test_gpu_parity.py tests/test_gpu_multi.py tests/test_gpu_edge.py tests/test_gpu_index.py -x -q > gpurun_out/pytest_lists.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_lists.log
timeout 900 python -m pytest tests/test_gpu_parity_large.py -x -q -k "c1" > gpurun_out/pytest_large_c1.log 2>&1; echo "large c1 rc=$?"; tail -3 gpurun_out/pytest_large_c1.log
python scripts/probe_drift.py c1 30 --stats-only > gpurun_out/probe_lists.log 2>&1; echo "probe rc=$?"; python - <<'PY'
import json
for l in open('gpurun_out/probe_lists.log'):
    if l.startswith('{'):
        d=json.loads(l); print(d['it'], round(d['ms'],3), 'upd', round(d['upd'],3), 'asg', round(d['asg'],3), 'scr', round(d['screen'],3), 'skip', d['skip_docs'], round(d['skip_ms'],3), 'moved', d['moved'], 'rec', d['recomputed'], 'th', round(d['theta'],4))
PY
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_lists.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_lists.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['iteration_ms']['warmup'], d['iteration_ms']['last_5_mean'], d['phase_ms'], d['drift_bound'], d['e2e']['value'], d['e2e']['wall_s'])"

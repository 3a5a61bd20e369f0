timeout 1200 python -m pytest tests/test_gpu_bound.py tests/test_gpu_parity.py tests/test_gpu_multi.py -x -q > gpurun_out/pytest_hash.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_hash.log
python scripts/probe_drift.py c1 34 --stats-only > gpurun_out/probe_t0.log 2>&1; python - <<'PY'
import json
rows=[json.loads(l) for l in open('gpurun_out/probe_t0.log') if l.startswith('{')]
m=lambda a,b,k: sum(d[k] for d in rows[a:b])/(b-a)
print('c1 adaptive', 'mean4-33 %.3f'%m(3,33,'ms'), 'last5 %.3f'%m(29,34,'ms'), [round(d['theta'],4) for d in rows])
PY
timeout 1500 python scripts/probe_drift.py c4 8 --stats-only > gpurun_out/probe_c4h.log 2>&1; echo "c4 rc=$?"; python - <<'PY'
import json
for l in open('gpurun_out/probe_c4h.log'):
    if l.startswith('{'):
        d=json.loads(l); print(d['it'], round(d['ms'],3), 'upd', round(d['upd'],3), 'asg', round(d['asg'],3), 'scr', round(d['screen'],3), 'skip', d['skip_docs'], 'exact', d['exact'], 'th', round(d['theta'],4), 'wall', round(d['wall'],2))
PY
tail -2 gpurun_out/probe_c4h.log | cut -c1-300
timeout 1200 python -m pytest tests/test_gpu_parity_large.py -x -q -k "c2 or c4" > gpurun_out/pytest_large_hash.log 2>&1; echo "large rc=$?"; tail -5 gpurun_out/pytest_large_hash.log

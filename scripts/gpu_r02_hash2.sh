timeout 1200 python -m pytest tests/test_gpu_bound.py -x -q > gpurun_out/pytest_hash2.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_hash2.log
for c in c2 c4 c3; do
timeout 1500 python scripts/probe_drift.py $c 12 --stats-only > gpurun_out/probe_${c}h2.log 2>&1; echo "$c rc=$?"; python - $c <<'PY'
import json,sys
for l in open(f'gpurun_out/probe_{sys.argv[1]}h2.log'):
    if l.startswith('{'):
        d=json.loads(l); print(d['it'], round(d['ms'],3), 'upd', round(d['upd'],3), 'asg', round(d['asg'],3), 'scr', round(d['screen'],3), 'skip', d['skip_docs'], 'exact', d['exact'], 'th', round(d['theta'],4), 'wall', round(d['wall'],2))
PY
done
timeout 1800 python -m pytest tests/test_gpu_sanitizer.py -x -q > gpurun_out/pytest_san.log 2>&1; echo "sanitizer rc=$?"; tail -30 gpurun_out/pytest_san.log | cut -c1-300

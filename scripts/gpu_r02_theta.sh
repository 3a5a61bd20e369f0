timeout 900 python -m pytest tests/test_gpu_bound.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_theta.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_theta.log
for t0 in 0.02 0.05; do
SSKM_THETA0=$t0 python scripts/probe_drift.py c1 34 --stats-only > gpurun_out/probe_theta_$t0.log 2>&1; echo "probe $t0 rc=$?"; python - $t0 <<'PY'
import json,sys
rows=[json.loads(l) for l in open(f'gpurun_out/probe_theta_{sys.argv[1]}.log') if l.startswith('{')]
for d in rows: print(d['it'], round(d['ms'],3), 'upd', round(d['upd'],3), 'asg', round(d['asg'],3), 'scr', round(d['screen'],3), 'skip', d['skip_docs'], 'moved', d['moved'], 'rec', d['recomputed'], 'th', round(d['theta'],4))
print('mean 4-33', sum(d['ms'] for d in rows[3:33])/30)
PY
done

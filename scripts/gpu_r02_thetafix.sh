for th in 0.003 0.006 0.012 0.025 0.05; do
SSKM_THETA=$th python scripts/probe_drift.py c1 34 --stats-only > gpurun_out/probe_fix_$th.log 2>&1; python - $th <<'PY'
import json,sys
rows=[json.loads(l) for l in open(f'gpurun_out/probe_fix_{sys.argv[1]}.log') if l.startswith('{')]
m=lambda a,b,k: sum(d[k] for d in rows[a:b])/(b-a)
print(sys.argv[1], 'mean4-33 %.3f'%m(3,33,'ms'), 'it4-8 %.3f'%m(3,8,'ms'), 'last5 %.3f'%m(29,34,'ms'), 'upd %.3f'%m(3,33,'upd'), 'scr %.3f'%m(3,33,'screen'), 'skip %.0f'%m(3,33,'skip_docs'))
PY
done
SSKM_HASH=1 timeout 900 python scripts/probe_drift.py c2 8 --stats-only > gpurun_out/probe_c2h.log 2>&1; echo "c2 rc=$?"; python - <<'PY'
import json
for l in open('gpurun_out/probe_c2h.log'):
    if l.startswith('{'):
        d=json.loads(l); print(d['it'], round(d['ms'],3), 'upd', round(d['upd'],3), 'asg', round(d['asg'],3), 'scr', round(d['screen'],3), 'skip', d['skip_docs'], 'exact', d['exact'], 'th', round(d['theta'],4))
PY
tail -3 gpurun_out/probe_c2h.log | cut -c1-300

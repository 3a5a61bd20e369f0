for c in c1 c3; do
timeout 900 python scripts/probe_drift.py $c 34 --stats-only > gpurun_out/probe_${c}t2.log 2>&1; echo "$c rc=$?"; python - $c <<'PY'
import json,sys
rows=[json.loads(l) for l in open(f'gpurun_out/probe_{sys.argv[1]}t2.log') if l.startswith('{')]
m=lambda a,b,k: sum(d[k] for d in rows[a:b])/(b-a)
print(sys.argv[1], 'mean4-33 %.3f'%m(3,33,'ms'), 'last5 %.3f'%m(29,34,'ms'), 'upd %.3f'%m(3,33,'upd'), 'scr %.3f'%m(3,33,'screen'), [round(d['theta'],4) for d in rows])
PY
done
timeout 1500 python scripts/probe_drift.py c4 10 --stats-only > gpurun_out/probe_c4t2.log 2>&1; echo "c4 rc=$?"; python - <<'PY'
import json
for l in open('gpurun_out/probe_c4t2.log'):
    if l.startswith('{'):
        d=json.loads(l); print(d['it'], round(d['ms'],3), 'upd', round(d['upd'],3), 'asg', round(d['asg'],3), 'scr', round(d['screen'],3), 'skip', d['skip_docs'], 'exact', d['exact'], 'th', round(d['theta'],4))
PY

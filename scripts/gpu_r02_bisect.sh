run() { python - "$@" <<'PY'
import json,os,subprocess,sys
label, cfg, iters = sys.argv[1], sys.argv[2], sys.argv[3]
env = dict(os.environ)
for kv in sys.argv[4:]:
    k, v = kv.split('='); env[k] = v
r = subprocess.run([sys.executable, 'scripts/probe_drift.py', cfg, iters, '--stats-only'], env=env, capture_output=True, text=True)
rows=[json.loads(l) for l in r.stdout.splitlines() if l.startswith('{')]
if not rows: print(label, 'FAILED', r.stderr[-500:]); sys.exit()
m=lambda a,b,k: sum(d[k] for d in rows[a:b])/max(1,(b-a))
n=len(rows)
print(label, cfg, 'mean4-%d %.3f'%(n, m(3,n,'ms')), 'last5 %.3f'%m(n-5,n,'ms'), 'upd %.3f'%m(3,n,'upd'), 'scr %.3f'%m(3,n,'screen'), 'ms', [round(d['ms'],1) for d in rows])
PY
}
for c in 608f75d faefe49 e80a42e; do run $c c3 14 SSKM_LIB=$PWD/paper_2108_00895_b200/lib_$c.so; done
run head c3 14

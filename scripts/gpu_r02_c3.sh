run() { # label env... config iters
python - "$@" <<'PY'
import json,os,subprocess,sys
label, cfg, iters = sys.argv[1], sys.argv[2], sys.argv[3]
env = dict(os.environ)
for kv in sys.argv[4:]:
    k, v = kv.split('='); env[k] = v
out = subprocess.run([sys.executable, 'scripts/probe_drift.py', cfg, iters, '--stats-only'], env=env, capture_output=True, text=True).stdout
rows=[json.loads(l) for l in out.splitlines() if l.startswith('{')]
m=lambda a,b,k: sum(d[k] for d in rows[a:b])/max(1,(b-a))
n=len(rows)
print(label, cfg, 'mean4-%d %.3f'%(n, m(3,n,'ms')), 'last5 %.3f'%m(n-5,n,'ms'), 'upd %.3f'%m(3,n,'upd'), 'scr %.3f'%m(3,n,'screen'), 'exact %.0f'%m(3,n,'exact'), 'th', [round(d['theta'],4) for d in rows[::4]])
PY
}
run default c3 16
run nokeep c3 16 SSKM_KEEP_LISTS=0
run noskip c3 16 SSKM_SKIP=0
run none c3 16 SSKM_SKIP=0 SSKM_KEEP_LISTS=0
run default c1 34
run nokeep c1 34 SSKM_KEEP_LISTS=0
run default c0 20
run default c2 10
run default c4 8

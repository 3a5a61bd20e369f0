# parity suite (PYTEST=1) + c1 bench + per-config probes: CFGS="c1:8 c3:8"
set -x
if [ -n "$PYTEST" ]; then timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log; fi
timeout 600 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_q.log 2>&1
tail -1 gpurun_out/bench_q.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('RESULT bench', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phase_ms'].items()}, round(d['roofline']['achieved'],1), d['roofline']['bytes_breakdown'])"
for cc in $CFGS; do c=${cc%%:*}; n=${cc##*:}
timeout 1500 python scripts/configs_probe.py $c ${MODE:-baseline} $n > gpurun_out/cfg_$c.log 2>&1; echo "$c rc=$?"
python -c "
import json
for l in open('gpurun_out/cfg_$c.log'):
    d=json.loads(l)
    if 'iter' in d: print('RESULT $c', d['iter'], d['ms'], d['update_ms'], d['screen_ms'], d['n_exact'], d['bound'])
"
done

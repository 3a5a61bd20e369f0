# quick GPU iteration: parity suite + c1 bench (+ optional extra command in $EXTRA)
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
CMD="python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline"
SSKM_DEBUG=1 timeout 600 $CMD > gpurun_out/plain.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/plain.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['phase_ms'], json.dumps(d['roofline'])[:700])"
grep sskm gpurun_out/plain.log | tail -3
if [ -n "$EXTRA" ]; then eval "$EXTRA"; fi

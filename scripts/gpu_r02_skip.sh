timeout 900 python -m pytest tests/test_gpu_bound.py tests/test_gpu_parity.py tests/test_gpu_multi.py -x -q > gpurun_out/pytest_skip.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_skip.log
timeout 900 python -m pytest tests/test_gpu_parity_large.py -x -q -k "c1" > gpurun_out/pytest_large_c1.log 2>&1; echo "large c1 rc=$?"; tail -3 gpurun_out/pytest_large_c1.log
python scripts/probe_drift.py c1 30 > gpurun_out/probe_drift2.log 2>&1; echo "probe rc=$?"; python - <<'PY'
import json
for l in open('gpurun_out/probe_drift2.log'):
    if l.startswith('{'):
        d=json.loads(l); print(d['it'], round(d['ms'],3), round(d['upd'],3), round(d['asg'],3), round(d['screen'],3), d['moved'], d['own'], d['exact'])
PY
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_skip.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_skip.log | cut -c1-1500

# parity suite on the default build, then the c1 bench on it and on scratch/lib_minb3.so
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
CMD="python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline"
show() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['phase_ms'], json.dumps(d['roofline']['bytes_breakdown']), d['roofline']['achieved'])"; }
SSKM_DEBUG=1 timeout 600 $CMD > gpurun_out/plain.log 2>&1; echo "bench rc=$?"; show gpurun_out/plain.log; grep sskm gpurun_out/plain.log | tail -2
cp -p paper_2108_00895_b200/libsskm_b200.so /tmp/lib_default.so
cp -p scratch/lib_minb3.so paper_2108_00895_b200/libsskm_b200.so
timeout 600 $CMD > gpurun_out/plain3.log 2>&1; echo "bench3 rc=$?"; show gpurun_out/plain3.log
cp -p /tmp/lib_default.so paper_2108_00895_b200/libsskm_b200.so

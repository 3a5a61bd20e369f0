# c1 bench on the in-tree build and on each prebuilt variant scratch/lib_*.so (loaded with SSKM_LIB);
# PYTEST=1 runs the GPU parity suite on the in-tree build first
set -x
if [ -n "$PYTEST" ]; then timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log; fi
CMD="python bench.py --steps ${STEPS:-10} --warmup 3 --no-e2e --no-cpu-baseline ${BENCH_ARGS}"
show() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('RESULT', '$2', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phase_ms'].items()}, round(d['roofline']['achieved'],1))"; }
for rep in ${REPS:-1}; do
timeout 600 $CMD > gpurun_out/v_default.log 2>&1; show gpurun_out/v_default.log default
for f in scratch/lib_*.so; do
  n=$(basename $f .so)
  SSKM_LIB=$PWD/$f timeout 600 $CMD > gpurun_out/v_$n.log 2>&1; show gpurun_out/v_$n.log $n
done
done

timeout 900 python -m pytest tests/test_gpu_bound.py tests/test_gpu_parity.py tests/test_gpu_edge.py -x -q > gpurun_out/s4_c4b_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s4_c4b_pytest.log
for r in 0.25 0.5; do
SSKM_SECOND_RATIO=$r SSKM_DEBUG=1 timeout 1500 python bench.py --config c4 --steps 9 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s4_c4b_$r.log 2> gpurun_out/s4_c4b_$r.err; echo "c4 ratio=$r rc=$?"; python - <<PY
import json
x=json.loads(open("gpurun_out/s4_c4b_$r.log").read().strip().splitlines()[-1])
print(x["ms_per_step"], x["iteration_ms"]["timed"], x["phase_ms"], x.get("exact_scan_docs_per_iter"))
PY
grep "second pass" gpurun_out/s4_c4b_$r.err | tail -2 | cut -c1-330
done

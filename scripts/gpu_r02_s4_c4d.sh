SSKM_DEBUG=1 timeout 1500 python bench.py --config c4 --steps 9 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s4_c4d.log 2> gpurun_out/s4_c4d.err; echo "c4 rc=$?"; python - <<PY
import json
x=json.loads(open("gpurun_out/s4_c4d.log").read().strip().splitlines()[-1])
print(x["ms_per_step"], x["iteration_ms"]["timed"], x["phase_ms"], x.get("exact_scan_docs_per_iter"))
PY
grep "second pass" gpurun_out/s4_c4d.err | tail -2 | cut -c1-330
timeout 2400 python -m pytest tests -m gpu -x -q --durations=6 > gpurun_out/s4_pytest2.log 2>&1; echo "pytest rc=$?"; tail -12 gpurun_out/s4_pytest2.log

timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_index.py tests/test_gpu_bound.py tests/test_gpu_multi.py -x -q > gpurun_out/s4_ncc_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s4_ncc_pytest.log
for m in baseline ncc; do
python scripts/configs_probe.py c1 $m 30 > gpurun_out/s4_c1_$m.log 2>&1; echo "$m rc=$?"
python - <<PY
import json
r=[json.loads(l) for l in open("gpurun_out/s4_c1_$m.log") if l.startswith('{"iter"')]
print("$m mean4-30", round(sum(x["ms"] for x in r[3:30])/27,3), "upd", round(sum(x["update_ms"] for x in r[3:30])/27,3), "asg", round(sum(x["assign_ms"] for x in r[3:30])/27,3), [x["ms"] for x in r[3:30:3]])
PY
done

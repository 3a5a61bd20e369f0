timeout 900 python -m pytest tests/test_gpu_bound.py tests/test_gpu_parity.py tests/test_gpu_edge.py -x -q > gpurun_out/s4_own2_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s4_own2_pytest.log
for rep in 1 2; do
python scripts/probe_drift.py c1 33 --stats-only > gpurun_out/s4_own2.log 2>&1; echo "rc=$?"
python - <<PY
import json
r=[json.loads(l) for l in open("gpurun_out/s4_own2.log") if l.startswith("{")]
print("mean4-33", round(sum(x["ms"] for x in r[3:33])/30,4), "upd", round(sum(x["upd"] for x in r[3:33])/30,4), "asg", round(sum(x["asg"] for x in r[3:33])/30,4), "screen", round(sum(x["screen"] for x in r[3:33])/30,4), "last5", round(sum(x["ms"] for x in r[28:33])/5,4))
print([round(x["screen"],3) for x in r[3:14]])
print("own", [x["own"] for x in r[3:33:4]], "gathers/own", [round(x["own_gathers"]/max(1,x["own"]),1) for x in r[3:33:4]])
PY
done

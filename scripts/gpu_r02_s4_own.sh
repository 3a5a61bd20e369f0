timeout 900 python -m pytest tests/test_gpu_bound.py tests/test_gpu_parity.py -x -q > gpurun_out/s4_own_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s4_own_pytest.log
for m in 0 1 2; do
SSKM_OWN_FIRST=$m python scripts/probe_drift.py c1 33 --stats-only > gpurun_out/s4_own_$m.log 2>&1; echo "own=$m rc=$?"
python - <<PY
import json
r=[json.loads(l) for l in open("gpurun_out/s4_own_$m.log") if l.startswith("{")]
print("mean4-33", sum(x["ms"] for x in r[3:33])/30, "screen", sum(x["screen"] for x in r[3:33])/30, "last5", sum(x["ms"] for x in r[28:33])/5)
for x in r[3:33:3]: print(x["it"], round(x["ms"],3), round(x["screen"],3), "visits",x["visits"],"own",x["own"],"ownonly",x["ownonly"],"skip",x["skip_docs"])
PY
done

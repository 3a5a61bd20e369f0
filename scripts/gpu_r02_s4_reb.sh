for late in 4 8 16; do
SSKM_REBUILD_LATE=$late python scripts/probe_drift.py c1 33 --stats-only > gpurun_out/s4_reb.log 2>&1; echo "late=$late rc=$?"
python - <<PY
import json
r=[json.loads(l) for l in open("gpurun_out/s4_reb.log") if l.startswith("{")]
print("mean4-33", round(sum(x["ms"] for x in r[3:33])/30,4), "upd", round(sum(x["upd"] for x in r[3:33])/30,4), "asg", round(sum(x["asg"] for x in r[3:33])/30,4), "screen", round(sum(x["screen"] for x in r[3:33])/30,4), "last5", round(sum(x["ms"] for x in r[28:33])/5,4), "last10", round(sum(x["ms"] for x in r[23:33])/10,4))
print([round(x["ms"],2) for x in r[13:33]])
PY
done

run() { python scripts/probe_drift.py c1 33 --stats-only > gpurun_out/s4_tmp.log 2>&1; python - <<PY
import json
r=[json.loads(l) for l in open("gpurun_out/s4_tmp.log") if l.startswith("{")]
print("$1: mean1-33", round(sum(x["ms"] for x in r[0:33])/33,4), "mean4-33", round(sum(x["ms"] for x in r[3:33])/30,4), "screen", round(sum(x["screen"] for x in r[3:33])/30,4), "last5", round(sum(x["ms"] for x in r[28:33])/5,4), [round(x["screen"],2) for x in r[0:10]], "theta", [round(x["theta"],4) for x in r[0:33:8]], "cand", [x["cand"] for x in r[3:33:8]], "exact", sum(x["exact"] for x in r))
PY
}
run default
SSKM_THETA0=0.0045 run theta0_0.0045
SSKM_THETA0=0.006 run theta0_0.006
SSKM_THETA0=0.009 run theta0_0.009
SSKM_THETA0=0.002 run theta0_0.002

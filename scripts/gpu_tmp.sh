run() { python scripts/probe_drift.py c1 20 --stats-only > gpurun_out/s4_tmp.log 2>&1; python - <<PY
import json
r=[json.loads(l) for l in open("gpurun_out/s4_tmp.log") if l.startswith("{")]
print("$1: mean4-20", round(sum(x["ms"] for x in r[3:20])/17,4), "asg", round(sum(x["asg"] for x in r[3:20])/17,4), "screen", round(sum(x["screen"] for x in r[3:20])/17,4), [round(x["screen"],3) for x in r[3:12]])
PY
}
run default
SSKM_L2_FETCH=32 run l2fetch32
SSKM_L2_FETCH=128 run l2fetch128
SSKM_SKIP=0 run noskip_index_order
SSKM_SKIP=0 SSKM_BOUND_ORDER=1 run noskip_cluster_order
SSKM_SKIP=0 SSKM_BOUND_ORDER=1 SSKM_L2_FETCH=32 run noskip_cluster_order_l2fetch32

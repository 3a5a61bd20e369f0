for lib in scratch/lib_mb5.so scratch/lib_mb3.so paper_2108_00895_b200/libsskm_b200.so; do
for rep in 1 2; do
SSKM_LIB=$PWD/$lib python scripts/probe_drift.py c1 33 --stats-only > gpurun_out/s4_lw.log 2>&1; echo "$lib rc=$?"
python - <<PY
import json
r=[json.loads(l) for l in open("gpurun_out/s4_lw.log") if l.startswith("{")]
print("mean4-33", round(sum(x["ms"] for x in r[3:33])/30,4), "upd", round(sum(x["upd"] for x in r[3:33])/30,4), "asg", round(sum(x["asg"] for x in r[3:33])/30,4), "screen", round(sum(x["screen"] for x in r[3:33])/30,4), "last5", round(sum(x["ms"] for x in r[28:33])/5,4), "it4-8 screen", [round(x["screen"],3) for x in r[3:8]])
PY
done; done

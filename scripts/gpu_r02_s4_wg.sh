for lib in scratch/lib_wg4.so scratch/lib_wg4_b12.so scratch/lib_wg4_b16.so scratch/lib_wg2_b16.so scratch/lib_wg3_b12.so; do
for rep in 1 2; do
SSKM_LIB=$PWD/$lib python scripts/probe_drift.py c1 33 --stats-only > gpurun_out/s4_wg.log 2>&1; echo "$lib rc=$?"
python - <<PY
import json
r=[json.loads(l) for l in open("gpurun_out/s4_wg.log") if l.startswith("{")]
print("mean4-33", round(sum(x["ms"] for x in r[3:33])/30,4), "upd", round(sum(x["upd"] for x in r[3:33])/30,4), "asg", round(sum(x["asg"] for x in r[3:33])/30,4), "screen", round(sum(x["screen"] for x in r[3:33])/30,4), "last5", round(sum(x["ms"] for x in r[28:33])/5,4), "upd it4-13", round(sum(x["upd"] for x in r[3:13])/10,4))
PY
done; done

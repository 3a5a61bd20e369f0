for f in 0.25 0; do
for c in c1 c3; do
SSKM_NCC_FULL_FRAC=$f python scripts/configs_probe.py $c ncc 30 > gpurun_out/s4_${c}_ncc_$f.log 2>&1; echo "$c frac=$f rc=$?"
python - <<PY
import json
r=[json.loads(l) for l in open("gpurun_out/s4_${c}_ncc_$f.log") if l.startswith('{"iter"')]
print("mean4-30", round(sum(x["ms"] for x in r[3:30])/27,3), "upd", round(sum(x["update_ms"] for x in r[3:30])/27,3), "asg", round(sum(x["assign_ms"] for x in r[3:30])/27,3), [x["ms"] for x in r[3:30:3]], [x["n_changed"] for x in r[3:30:3]])
PY
done; done

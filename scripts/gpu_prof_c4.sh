set -x
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bound_screen_kernel" -s 3 -c 1 -o gpurun_out/prof_bound5 $CMD > gpurun_out/ncu_prof_bound5.log 2>&1; echo "ncu rc=$?"
timeout 900 ncu --set full --clock-control none -k regex:"hipost_build_kernel|write_cols_kernel" -s 6 -c 2 -o gpurun_out/prof_upd $CMD > gpurun_out/ncu_prof_upd.log 2>&1; echo "ncu2 rc=$?"
timeout 1500 python scripts/configs_probe.py c4 baseline 5 > gpurun_out/cfg_c4.log 2>&1; echo "c4 rc=$?"
python -c "
import json
for l in open('gpurun_out/cfg_c4.log'):
    d=json.loads(l)
    if 'iter' in d: print('RESULT c4', d['iter'], d['ms'], d['update_ms'], d['screen_ms'], d['n_exact'], d['bound'])
"

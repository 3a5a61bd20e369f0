set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bound_screen_kernel" -s 3 -c 1 -o gpurun_out/prof_c3 python scripts/configs_probe.py c3 baseline 5 > gpurun_out/ncu_c3.log 2>&1; echo "rc=$?"

set -x
python scripts/prof_one.py c1 2 > gpurun_out/p1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"^postings_screen" -s 2 -c 1 -o gpurun_out/prof_post python scripts/prof_one.py c1 2 > gpurun_out/ncu_s1.log 2>&1
echo "rc=$?"

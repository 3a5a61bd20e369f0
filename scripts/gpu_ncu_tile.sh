set -x
export SSKM_SCREEN_UNROLL=16 SSKM_TILE_BYTES=134217728 SSKM_ORDER=0
python scripts/prof_one.py c1 2 > gpurun_out/p1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"^screen_tile" -s 10 -c 1 -o gpurun_out/prof_screen128 python scripts/prof_one.py c1 2 > gpurun_out/ncu_s1.log 2>&1
echo "rc=$?"
export SSKM_SCREEN_UNROLL=8 SSKM_TILE_BYTES=67108864 SSKM_ORDER=1
python scripts/prof_one.py c1 2 > gpurun_out/p2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"^screen_tile|^resolve" -s 20 -c 2 -o gpurun_out/prof_screen64 python scripts/prof_one.py c1 2 > gpurun_out/ncu_s2.log 2>&1
echo "rc=$?"

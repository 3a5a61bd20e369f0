set -x
for kt in 512 1024; do
SSKM_POST_KT=$kt timeout 900 python scripts/configs_probe.py c4 baseline 1 > gpurun_out/cfg_c4_$kt.log 2>&1; echo "c4 kt=$kt rc=$?"; tail -1 gpurun_out/cfg_c4_$kt.log
SSKM_POST_KT=$kt timeout 900 python scripts/configs_probe.py c2 baseline 3 > gpurun_out/cfg_c2_$kt.log 2>&1; echo "c2 kt=$kt rc=$?"; tail -1 gpurun_out/cfg_c2_$kt.log
SSKM_POST_KT=$kt timeout 900 python scripts/configs_probe.py c1 baseline 5 > gpurun_out/cfg_c1_$kt.log 2>&1; echo "c1 kt=$kt rc=$?"; tail -1 gpurun_out/cfg_c1_$kt.log
done

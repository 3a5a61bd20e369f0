timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "kmeanspp" > gpurun_out/pytest_kpp.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_kpp.log
timeout 600 python scripts/probe_kpp.py c1; SSKM_KPP_HOST=1 timeout 600 python scripts/probe_kpp.py c1
timeout 900 python scripts/probe_kpp.py c2

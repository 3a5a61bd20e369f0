timeout 900 python -m pytest tests/test_vectorize.py -x -q > gpurun_out/vec_tests.log 2>&1; echo "vec tests rc=$?"; tail -15 gpurun_out/vec_tests.log
timeout 900 python scripts/bench_vectorize.py 20000 200000 500000 > gpurun_out/vec_bench.log 2>&1; echo "vec bench rc=$?"; cat gpurun_out/vec_bench.log | tail -5

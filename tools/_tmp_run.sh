timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_engine.py -x -q -m gpu > gpurun_out/q63_pytest.log 2>&1; tail -1 gpurun_out/q63_pytest.log
bash tools/ab_lib.sh q63 "c2 c4" "base prev base prev"

timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/q69_pytest.log 2>&1; tail -1 gpurun_out/q69_pytest.log
FMM2D_LIBRARY=build/ab/libfmm2d_fnone.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_engine.py -x -q -m gpu > gpurun_out/q69_pytest2.log 2>&1; tail -1 gpurun_out/q69_pytest2.log
bash tools/ab_lib.sh q69 "c5 c2" "base fall fnone"

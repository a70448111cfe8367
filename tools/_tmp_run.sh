FMM2D_LIBRARY=build/ab/libfmm2d_ke0.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_engine.py -x -q -m gpu > gpurun_out/q67_pytest.log 2>&1; tail -1 gpurun_out/q67_pytest.log
bash tools/ab_lib.sh q67 "c5 c2 c3" "base ke0 ke2"

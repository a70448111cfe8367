timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/q71_pytest.log 2>&1; tail -1 gpurun_out/q71_pytest.log
bash tools/ab_lib.sh q71 "c5 c2" "base old"

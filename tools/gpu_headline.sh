#!/bin/bash
# Headline-config parity (C2-C5 vs reference goldens) + the full GPU suite + one C2 bench line.
TAG=${1:-h}
O=gpurun_out/$TAG; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_headline.py -x -q -s -m gpu > $O/pytest_headline.log 2>&1; echo "rc=$?" >> $O/pytest_headline.log
tail -15 $O/pytest_headline.log
timeout 900 python -m pytest tests -x -q -m gpu --deselect tests/test_gpu_headline.py > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
timeout 300 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c2.json 2> $O/bench_c2.err
tail -c 600 $O/bench_c2.json

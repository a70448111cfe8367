#!/bin/bash
# Quick GPU iteration: gpu tests, C2 bench, optional ncu capture of a kernel regex.
# Usage (inside gpurun): bash tools/gpu_quick.sh TAG [kernel_regex] [config]
TAG=${1:-q}; KRE=${2:-}; CFG=${3:-c2}
O=gpurun_out/$TAG; mkdir -p $O
timeout 900 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
timeout 300 python bench.py --config $CFG --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_$CFG.json 2> $O/bench_$CFG.err
python -c "import json;d=json.load(open('$O/bench_$CFG.json'));print(d['ms_per_step'],d['phase_ms'],d['roofline']['frac'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
if [ -n "$KRE" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KRE" -c 2 \
  -o $O/prof python bench.py --config $CFG --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_full.log 2>&1
fi
echo done

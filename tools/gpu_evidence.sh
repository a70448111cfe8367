#!/bin/bash
# HEAD evidence in one gpurun call: full GPU suite, smoke, bench C1-C5, reference arm, launch lists.
# Usage (inside gpurun): bash tools/gpu_evidence.sh <tag>
TAG=${1:-ev}
O=gpurun_out/$TAG; mkdir -p $O
nvidia-smi > $O/nvidia-smi.txt 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
for c in c2 c3 c4 c5 c1; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err
  tail -c 300 $O/bench_$c.json
done
if [ "${REF:-1}" = 1 ]; then
timeout 400 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
fi
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv \
  python bench.py --config c2 --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c5.csv \
  python bench.py --config c5 --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
echo done

#!/bin/bash
# One gpurun call: GPU tests, smoke, bench lines, launch list, ncu captures.
# Usage (inside gpurun): bash tools/gpu_round.sh [tag]
TAG=${1:-r01}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi > $O/nvidia-smi.txt 2>&1
cat MEASURED_PEAKS.json > $O/measured_peaks.json 2>/dev/null
timeout 900 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
for c in c2 c3 c4 c5 c1; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv \
  python bench.py --config c2 --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c5.csv \
  python bench.py --config c5 --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_m2l_dense|k_p2p' -c 2 \
  -o $O/prof_c2 python bench.py --config c2 --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_part_step|k_subtree|k_classify|k_reclassify|k_l2p|k_p2l' -s 12 -c 8 \
  -o $O/prof_c2_rest python bench.py --config c2 --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_full2.log 2>&1
echo done

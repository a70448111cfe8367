#!/bin/bash
# M2L contraction-blocking A/B (library variants) + ncu --set full of the tree kernels at C2 and C5.
TAG=${1:-abt}
O=gpurun_out/$TAG; mkdir -p $O
bash tools/ab_lib.sh $TAG "c2 c4 c5" "base jb2 jb3 jb2w12"
KRE='k_bbox|k_make_keys|DeviceRadixSort|k_fix_ties|k_part_step|k_subtree|k_gather_points|k_init_arrays'
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KRE" -c 24 \
  -o $O/tree_c2 python bench.py --config c2 --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_c2.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$KRE" -c 30 \
  -o $O/tree_c5 python bench.py --config c5 --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_c5.log 2>&1
echo done

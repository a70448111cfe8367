#!/bin/bash
# P2P seed probe + A/B (MUFU vs soft seed), ncu of the tree kernels (C2, C5) and P2P (C5):
# reports are exported to raw CSV + per-launch summaries on the box and deleted (size cap).
TAG=${1:-seed}
O=gpurun_out/$TAG; mkdir -p $O
./tools/p2p_mix > $O/p2p_mix.json 2>&1; cat $O/p2p_mix.json
bash tools/ab_lib.sh $TAG "c2 c5" "base soft"
FMM2D_LIBRARY=build/ab/libfmm2d_soft.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_headline.py -x -q -m gpu > $O/pytest_soft.log 2>&1; echo "rc=$?" >> $O/pytest_soft.log
tail -2 $O/pytest_soft.log
KRE='k_bbox|k_make_keys|DeviceRadixSort|k_fix_ties|k_part_step|k_subtree|k_gather_points|k_init_arrays'
prof() {  # name config kernel-regex count
  timeout 1200 ncu --set full --clock-control none -k regex:"$3" -c $4 -o $O/$1 \
    python bench.py --config $2 --steps 1 --warmup 0 --no-cpu-baseline > $O/$1.log 2>&1
  ncu -i $O/$1.ncu-rep --page raw --csv > $O/$1_raw.csv 2>/dev/null
  python tools/ncu_multi.py $O/$1.ncu-rep > $O/$1_summary.txt 2>&1
  rm -f $O/$1.ncu-rep
}
prof tree_c2 c2 "$KRE" 24
prof tree_c5 c5 "$KRE" 30
prof p2p_c5 c5 'k_p2p' 1
FMM2D_LIBRARY=build/ab/libfmm2d_soft.so prof p2p_c5_soft c5 'k_p2p' 1
du -sh $O
echo done

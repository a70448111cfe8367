#!/bin/bash
# M2L immediate-coefficient A/B: parity of the variant, bench C2-C5, ncu of M2L (summaries only).
TAG=${1:-imm}
O=gpurun_out/$TAG; mkdir -p $O
FMM2D_LIBRARY=build/ab/libfmm2d_imm.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_headline.py -x -q -m gpu > $O/pytest_imm.log 2>&1; echo "rc=$?" >> $O/pytest_imm.log
tail -2 $O/pytest_imm.log
bash tools/ab_lib.sh $TAG "c2 c3 c4 c5" "base imm"
prof() {  # name config kernel-regex count
  timeout 900 ncu --set full --clock-control none -k regex:"$3" -c $4 -o $O/$1 \
    python bench.py --config $2 --steps 1 --warmup 0 --no-cpu-baseline > $O/$1.log 2>&1
  ncu -i $O/$1.ncu-rep --page raw --csv > $O/$1_raw.csv 2>/dev/null
  python tools/ncu_multi.py $O/$1_raw.csv > $O/$1_summary.txt 2>&1
  rm -f $O/$1.ncu-rep
}
prof m2l_c2_base c2 'k_m2l_dense' 1
FMM2D_LIBRARY=build/ab/libfmm2d_imm.so prof m2l_c2_imm c2 'k_m2l_dense' 1
cat $O/m2l_c2_base_summary.txt $O/m2l_c2_imm_summary.txt | cut -c1-220
echo done

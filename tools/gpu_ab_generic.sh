#!/bin/bash
# Generic library-variant A/B: parity tests on the variant, then bench configs.
#   bash tools/gpu_ab_generic.sh TAG VARIANT "c1 c2 c5"
TAG=$1; V=$2; CFGS=${3:-"c1 c2 c3 c5"}
O=gpurun_out/$TAG; mkdir -p $O
FMM2D_LIBRARY=build/ab/libfmm2d_$V.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_engine.py tests/test_gpu_headline.py -x -q -m gpu > $O/pytest_$V.log 2>&1; echo "rc=$?" >> $O/pytest_$V.log
tail -2 $O/pytest_$V.log
bash tools/ab_lib.sh $TAG "$CFGS" "base $V"
echo done

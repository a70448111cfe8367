#!/bin/bash
# GPU suite with the default build, then an env-switch A/B: bash tools/gpu_ab_env.sh TAG VAR=a,b "c1 c2"
TAG=$1; SPEC=$2; CFGS=${3:-"c1 c2 c3 c5"}
O=gpurun_out/$TAG; mkdir -p $O
timeout 1200 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
for c in $CFGS; do bash tools/ab.sh $TAG $c $SPEC; done
echo done

#!/bin/bash
# A/B of library variants (build/ab/libfmm2d_NAME.so, "base" = in-tree build):
#   bash tools/ab_lib.sh TAG "c2 c5" "base v1 v2"
TAG=$1; CFGS=$2; VARS=$3
O=gpurun_out/$TAG; mkdir -p $O
for cfg in $CFGS; do
  for v in $VARS; do
    f=$O/${cfg}_$v.json
    if [ $v = base ]; then
      timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline > $f 2>&1
    else
      FMM2D_LIBRARY=build/ab/libfmm2d_$v.so timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline > $f 2>&1
    fi
    echo "$cfg $v $(python -c "import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);print(round(d['ms_per_step'],4),'e2e',round(d['e2e']['ms_per_step'],4),d['phase_ms'])" 2>&1 | tail -1)"
  done
done

#!/bin/bash
# A/B of env-selected variants on one config: bash tools/ab.sh TAG CONFIG VAR=val1,val2,...
TAG=$1; CFG=$2; SPEC=$3
O=gpurun_out/$TAG; mkdir -p $O
VAR=${SPEC%%=*}; VALS=${SPEC#*=}
for v in ${VALS//,/ }; do
  f=$O/ab_${CFG}_${VAR}_$(echo $v | tr '/.' '__').json
  env $VAR=$v timeout 300 python bench.py --config $CFG --steps 10 --warmup 3 --no-cpu-baseline > $f 2>&1
  echo "$CFG $VAR=$v $(python -c "import json;d=json.load(open('$f'));print(round(d['ms_per_step'],4),d['phase_ms'])" 2>&1 | tail -1)"
done

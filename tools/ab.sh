#!/bin/bash
# A/B of env-selected variants on one config: bash tools/ab.sh TAG CONFIG VAR=val1,val2,...
TAG=$1; CFG=$2; SPEC=$3
O=gpurun_out/$TAG; mkdir -p $O
VAR=${SPEC%%=*}; VALS=${SPEC#*=}
for v in ${VALS//,/ }; do
  env $VAR=$v timeout 300 python bench.py --config $CFG --steps 10 --warmup 3 --no-cpu-baseline > $O/ab_${VAR}_$v.json 2>&1
  echo "$VAR=$v $(python -c "import json;d=json.load(open('$O/ab_${VAR}_$v.json'));print(round(d['ms_per_step'],4),d['phase_ms'])")"
done

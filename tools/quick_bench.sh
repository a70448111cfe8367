#!/bin/bash
# quick check: GPU parity + engine tests, bench lines (phase times), optional ncu of a kernel
TAG=${1:-q}; KRE=${2:-}; CFGS=${3:-"c2 c3 c5"}
O=gpurun_out/$TAG; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_engine.py tests/test_gpu_headline.py -x -q -m gpu > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
tail -2 $O/pytest.log
for c in $CFGS; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $O/$c.json 2> $O/$c.err
  echo "$c $(python -c "import json;d=json.loads(open('$O/$c.json').read().strip().splitlines()[-1]);print(round(d['ms_per_step'],4),'e2e',round(d['e2e']['ms_per_step'],4),{k:round(v,4) for k,v in d['phase_ms'].items()})")"
done
if [ -n "$KRE" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KRE" -c 1 \
  -o $O/prof python bench.py --config c2 --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu.log 2>&1
fi
echo done

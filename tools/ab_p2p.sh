#!/bin/bash
# P2P A/B: GPU parity tests with the default build, library variants on the
# headline configs, the P2P-beside-M2L overlap switch, the C5 error probe per
# variant, and an ncu capture of the default P2P kernel.
TAG=${1:-p2p}; VARS=${2:-"base nofast"}; PROBE=${3:-"base"}
O=gpurun_out/$TAG; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_engine.py -x -q -m gpu > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
tail -2 $O/pytest.log
bash tools/ab_lib.sh $TAG "c2 c3 c5" "$VARS"
for c in c2 c5; do
  FMM2D_P2P_OVERLAP=0 timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $O/${c}_noovl.json 2>&1
  echo "$c no-overlap $(python -c "import json;d=json.loads(open('$O/${c}_noovl.json').read().strip().splitlines()[-1]);print(round(d['ms_per_step'],4),d['phase_ms'])")"
done
for v in $PROBE; do
  if [ $v = base ]; then timeout 600 python tools/c5_error_probe.py; else FMM2D_LIBRARY=build/ab/libfmm2d_$v.so timeout 600 python tools/c5_error_probe.py; fi
done
FMM2D_P2P_OVERLAP=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_p2p' -c 1 \
  -o $O/prof_c2 python bench.py --config c2 --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu.log 2>&1
echo done

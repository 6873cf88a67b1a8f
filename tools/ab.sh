#!/bin/bash
# A/B the experimental library builds under exp/ on one workload.
WL=${1:-C4s}; STEPS=${2:-20}
for d in exp/*/; do
  v=$(basename $d)
  SILT_LIB=$d/libsilt_b200.so python bench.py --workload $WL --steps $STEPS --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys
try:
  d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],4), 'ms', round(d['value']/1e9,3), 'Gcell/s')
except Exception as e: print('$v failed', e)"
done

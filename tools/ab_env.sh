#!/bin/bash
# A/B one build under different environment settings: ab_env.sh WL STEPS "ENV1" "ENV2" ...
WL=$1; STEPS=$2; shift 2
for e in "$@"; do
  env $e python bench.py --workload $WL --steps $STEPS --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys
try:
  d=json.loads(sys.stdin.read()); print('$e', round(d['ms_per_step'],4), 'ms', round(d['value']/1e9,3), 'Gcell/s')
except Exception as ex: print('$e failed', ex)"
done

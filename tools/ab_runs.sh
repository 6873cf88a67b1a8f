#!/bin/bash
# A/B of the builds under exp/*/ (exp/base = reference build): bitwise field comparison
# (tools/bitcmp.py) and bench timings.  usage: tools/ab_runs.sh TAG [WORKLOADS]  -> gpurun_out/ab_TAG.log
TAG=$1
WLS=${2:-"C5:100 C3:300 C4:20"}
OUT=gpurun_out/ab_$TAG.log
: > $OUT
for d in exp/*/; do
  v=$(basename $d); [ "$v" = base ] && continue
  echo "== bitcmp base vs $v" >> $OUT
  timeout 600 python tools/bitcmp.py exp/base/libsilt_b200.so $d/libsilt_b200.so >> $OUT 2>&1
done
for WL in $WLS; do
  W=${WL%%:*}; K=${WL##*:}
  echo "== $W $K" >> $OUT
  for rep in 1 2; do
  for d in exp/*/; do
    v=$(basename $d)
    SILT_LIB=$d/libsilt_b200.so timeout 600 python bench.py --workload $W --steps $K --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys
try:
  d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],4), 'ms', round(d['value']/1e9,3), 'Gcell/s', d.get('clocks',{}).get('sm_mhz'))
except Exception as e: print('$v failed', e)" >> $OUT
  done
  done
done
cat $OUT

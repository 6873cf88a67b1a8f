#!/bin/bash
# Round-end measurement set (one GPU): bench lines, launch list, ncu --set full of one step
# launch per workload.  Outputs under gpurun_out/rf_*; summarised into profiles/r2_* by
# tools/profile_summary.py (see profiles/README.md).
set -x
O=gpurun_out
python bench.py --steps 20 --warmup 5 > $O/rf_bench_c4.json 2> $O/rf_bench.err
python bench.py --steps 500 --warmup 5 --no-cpu-baseline > $O/rf_bench_c4_500.json 2>> $O/rf_bench.err
python bench.py --workload C5 --steps 300 > $O/rf_bench_c5.json 2>> $O/rf_bench.err
python bench.py --workload C3 --steps 1000 > $O/rf_bench_c3.json 2>> $O/rf_bench.err
python bench.py --workload Q --steps 100 --no-cpu-baseline > $O/rf_bench_q.json 2>> $O/rf_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/rf_launches_c4.csv \
    python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > $O/rf_ncu_launches.log 2>&1
for WL in C4 Q C5; do
  ncu --set full --import-source on --clock-control none -k regex:step2d_kernel -s 3 -c 1 -o $O/rf_full_$WL \
      python bench.py --workload $WL --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/rf_ncu_full_$WL.log 2>&1
done
# C3's 32 MB state stays in L2 across steps: no cache flush, so DRAM counts are the kernel's own
ncu --set full --import-source on --clock-control none --cache-control none -k regex:step2d_kernel -s 600 -c 1 \
    -o $O/rf_full_C3 python bench.py --workload C3 --steps 2 --warmup 600 --no-e2e --no-cpu-baseline \
    > $O/rf_ncu_full_C3.log 2>&1
ls -la $O/rf_*

#!/bin/bash
# Round-end measurement set (one GPU): bench lines, launch list, ncu --set full of one step
# launch per workload, CTA timeline.  Outputs under gpurun_out/; summarised into profiles/
# by tools/profile_summary.py.
set -x
python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
python bench.py --workload C5 --steps 300 > gpurun_out/bench_c5.json 2>> gpurun_out/bench_c4.err
python bench.py --workload Q --steps 100 --no-cpu-baseline > gpurun_out/bench_q.json 2>> gpurun_out/bench_c4.err
python bench.py --workload C4 --steps 50 --no-cpu-baseline > gpurun_out/bench_c4_50.json 2>> gpurun_out/bench_c4.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c4.csv \
    python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
for WL in C4 Q C5; do
  ncu --set full --import-source on --clock-control none -k regex:step2d_kernel -s 3 -c 1 -o gpurun_out/full_$WL \
      python bench.py --workload $WL --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_$WL.log 2>&1
done
SILT_LIB=exp/trace/libsilt_b200.so python tools/cta_trace.py C4 499 gpurun_out/trace_c4_499.npz > gpurun_out/trace_c4.log 2>&1
SILT_LIB=exp/trace/libsilt_b200.so python tools/cta_trace.py C4 5 gpurun_out/trace_c4_5.npz >> gpurun_out/trace_c4.log 2>&1

#!/bin/bash
# C4 throughput under each Shields law (profiles/r1_shields_bench.md)
python bench.py --steps 20 --warmup 5 --no-e2e > gpurun_out/shields_grass.json 2>/dev/null
for law in camenen:manning flvb:manning mpm:darcy-weisbach mpm:manning nielsen:darcy-weisbach ribberink:manning; do
  python bench.py --steps 20 --warmup 5 --law $law --no-e2e > gpurun_out/shields_${law/:/_}.json 2>/dev/null
done

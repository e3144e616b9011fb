#!/bin/bash
# Refresh the per-config bench lines under gpurun_out/ (copied to profiles/r01_bench_*.json).
set -u
mkdir -p gpurun_out
for cfg in C1 C2 C3 C3dc C4g DM14; do
  timeout 600 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/bench_$cfg.json
done
for p in 2 4 8; do
  timeout 600 python bench.py --virtual-shards $p --steps 2 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/bench_virtual_shards_$p.json
done
timeout 600 python bench.py --precision c64 --steps 3 --warmup 3 --no-cpu-baseline --no-grad 2>/dev/null | tail -1 > gpurun_out/bench_c64.json
echo done

#!/bin/bash
# A/B of gradient builds: abtest/libsv_<v>.so per argument, two interleaved rounds of
# tools/experiments/ab_da_cost.py (default plan, fixed parameters) on C2, C3 and C4g.
for r in 1 2; do
  for v in "$@"; do
    cp abtest/libsv_$v.so paper_2406_17248_b200/libsv.so
    echo "$v $(for c in C2 C3 C4g; do python tools/experiments/ab_da_cost.py $c -1 | awk '{print $3}'; done | tr '\n' ' ')"
  done
done

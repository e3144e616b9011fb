#!/bin/bash
# A/B of forward builds: abtest/libsv_<v>.so for each argument, two interleaved rounds, the best
# steady-state circuit time of tools/prof_pass.py 30 40 (the C4 generator) per run.
for r in 1 2; do
  for v in "$@"; do
    cp abtest/libsv_$v.so paper_2406_17248_b200/libsv.so
    echo "$v $(python tools/prof_pass.py 30 40 | grep iter | sort -t: -k2 -n | awk '{print $3}' | sort -n | head -1)"
  done
done

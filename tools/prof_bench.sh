#!/bin/bash
# Round evidence (run under gpurun from the repo root): the bench line, the ncu launch list of the
# same command, and one `ncu --set full` capture of the dominant kernel (a 30-qubit forward pass).
set -u
mkdir -p gpurun_out
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench_rc=$?"
tail -1 gpurun_out/bench.json
# launch list (cold-cache, serialised: compare shares, not absolutes)
python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-grad > gpurun_out/plain_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-grad > gpurun_out/ncu_launches.log 2>&1
echo "launches_rc=$?"
# full capture of one steady-state forward pass at 30q
python tools/prof_pass.py 30 40 > gpurun_out/prof30_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_pass -s 70 -c 1 \
    -o gpurun_out/prof_pass30 python tools/prof_pass.py 30 40 > gpurun_out/ncu_full.log 2>&1
echo "full_rc=$?"

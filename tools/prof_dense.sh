#!/bin/bash
# ncu --set full capture of one steady-state all-dense forward pass (k_pass_dense) at 30 qubits.
set -u
mkdir -p gpurun_out
python tools/prof_pass.py 30 40 > gpurun_out/prof_dense_plain.log 2>&1; echo "plain_rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_pass_dense -s 20 -c 1 \
    -o gpurun_out/prof_dense python tools/prof_pass.py 30 40 > gpurun_out/ncu_dense.log 2>&1
echo "ncu_rc=$?"

#!/bin/bash
# ncu --set full capture of the heaviest C4g adjoint pass (the 8th DUAL launch: adjoint dense stages
# plus sequential register stages).
set -u
mkdir -p gpurun_out
python tools/prof_config.py C4g 1 > gpurun_out/prof_dual_plain.log 2>&1; echo "plain_rc=$?"
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_pass_reg<\(int\)3, \(bool\)1>' -s 7 -c 1 \
    -o gpurun_out/prof_dual_da python tools/prof_config.py C4g 1 > gpurun_out/ncu_dual_da.log 2>&1
echo "ncu_rc=$?"

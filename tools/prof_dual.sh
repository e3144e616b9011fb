#!/bin/bash
# ncu --set full capture of adjoint (DUAL) passes of the C4g gradient evaluation.
set -u
mkdir -p gpurun_out
python tools/prof_config.py C4g 1 > gpurun_out/prof_dual_plain.log 2>&1; echo "plain_rc=$?"
SV_PLAN_DEBUG=1 python tools/prof_config.py C4g 1 > gpurun_out/prof_dual_plan.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_pass_reg<\(int\)3, \(bool\)1>' -c 3 \
    -o gpurun_out/prof_dual python tools/prof_config.py C4g 1 > gpurun_out/ncu_dual.log 2>&1
echo "ncu_rc=$?"

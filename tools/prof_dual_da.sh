#!/bin/bash
# ncu --set full captures of C4g adjoint passes: the heaviest one with adjoint dense stages (the 4th
# launch of the general instantiation k_pass_reg<3, true, false>) and one sequential pass of the
# single-buffered instantiation k_pass_reg<3, true, true>.
set -u
mkdir -p gpurun_out
python tools/prof_config.py C4g 1 > gpurun_out/prof_dual_plain.log 2>&1; echo "plain_rc=$?"
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:k_pass_reg<\(int\)3, \(bool\)1, \(bool\)0' -s 3 -c 1 \
    -o gpurun_out/prof_dual_da python tools/prof_config.py C4g 1 > gpurun_out/ncu_dual_da.log 2>&1
echo "ncu_da_rc=$?"
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:k_pass_reg<\(int\)3, \(bool\)1, \(bool\)1>' -s 1 -c 1 \
    -o gpurun_out/prof_dual_sb python tools/prof_config.py C4g 1 > gpurun_out/ncu_dual_sb.log 2>&1
echo "ncu_sb_rc=$?"

#!/bin/bash
# Round-2 evidence batch (run under gpurun from the repo root): GPU tests, smoke, every bench line,
# the ncu launch list of the default bench command and full captures of the dominant kernels.
set -x
O=gpurun_out/${R02_OUT:-r02f}
mkdir -p $O
python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
python bench.py > $O/bench.json 2> $O/bench.err
for c in C1 C2 C3 C3dc C4g DM14; do python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err; done
python bench.py --precision c64 > $O/bench_c64.json 2> $O/bench_c64.err
for v in 2 4 8; do python bench.py --virtual-shards $v > $O/bench_vs$v.json 2> $O/bench_vs$v.err; done
python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
# launch list of the default bench command (cold-cache, serialised: compare shares)
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-grad > $O/ncu_launches.log 2>&1
# full captures: forward dense pass, complex64 pass, heaviest C4g adjoint pass
ncu --set full --clock-control none --import-source on -k regex:k_pass_dense -s 20 -c 1 \
    -o $O/prof_dense python tools/prof_pass.py 30 40 > $O/ncu_dense.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_pass_c64 -s 20 -c 1 \
    -o $O/prof_c64 python bench.py --precision c64 --no-cpu-baseline --no-grad --steps 1 --warmup 1 > $O/ncu_c64.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:k_pass_reg<\(int\)3, \(bool\)1, \(bool\)0' -s 3 -c 1 -o $O/prof_dual_da python tools/prof_config.py C4g 1 > $O/ncu_dual_da.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_pauli_tile -s 3 -c 1 \
    -o $O/prof_pauli python tools/prof_config.py C4g 1 > $O/ncu_pauli.log 2>&1
echo done

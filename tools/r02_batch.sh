set -x
mkdir -p gpurun_out/r02
python -m pytest tests -m gpu -x -q > gpurun_out/r02/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02/smoke.log 2>&1
python bench.py > gpurun_out/r02/bench.json 2> gpurun_out/r02/bench.err
for c in C1 C2 C3 C3dc C4g DM14; do python bench.py --config $c > gpurun_out/r02/bench_$c.json 2> gpurun_out/r02/bench_$c.err; done
python bench.py --precision c64 > gpurun_out/r02/bench_c64.json 2> gpurun_out/r02/bench_c64.err
for v in 2 4 8; do python bench.py --virtual-shards $v > gpurun_out/r02/bench_vs$v.json 2> gpurun_out/r02/bench_vs$v.err; done
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r02/bench_ref.json 2> gpurun_out/r02/bench_ref.err

for cfg in C1 C2 C3 C3dc C4g; do
  timeout 600 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/bench_$cfg.json
done

for v in 96 150 250 400; do
  SV_DA_MIN_COST=$v timeout 300 python bench.py --config C3 --steps 4 --warmup 3 --no-cpu-baseline 2>&1 | python -c "import sys,json
for l in sys.stdin:
  if l.startswith('{'): d=json.loads(l); print('C3 mincost=$v', round(d['value'],2), round(d['fixed_params_value'],2))" >> gpurun_out/exp_c3cost.txt
done

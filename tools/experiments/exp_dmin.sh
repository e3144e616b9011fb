for v in 20 8 1; do
  SV_DENSE_MIN_COST=$v timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-grad 2>&1 | python -c "import sys,json
for l in sys.stdin:
  if l.startswith('{'): d=json.loads(l); print('C4 dmin=$v', round(d['value'],1))" >> gpurun_out/exp_dmin.txt
done

for v in 6 5 4; do
  echo "== SV_DENSE_MAX_VAR=$v" >> gpurun_out/exp_maxvar.txt
  SV_DENSE_MAX_VAR=$v python tools/experiments/exp_replan.py C2 C3 >> gpurun_out/exp_maxvar.txt 2>&1
  SV_DENSE_MAX_VAR=$v timeout 300 python bench.py --steps 2 --warmup 2 --no-cpu-baseline --no-grad 2>&1 | python -c "import sys,json
for l in sys.stdin:
  if l.startswith('{'): d=json.loads(l); print('C4', round(d['value'],1))" >> gpurun_out/exp_maxvar.txt
done

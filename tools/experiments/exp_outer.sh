for v in "0 96" "1 96" "2 200" "1 200" "2 400"; do
  set -- $v
  for cfg in C3 C4g; do
    SV_DA_MAX_OUTER=$1 SV_DA_MIN_COST=$2 timeout 300 python bench.py --config $cfg --steps 3 --warmup 2 --no-cpu-baseline 2>&1 | python -c "import sys,json
for l in sys.stdin:
  if l.startswith('{'): d=json.loads(l); print('$cfg outer=$1 mincost=$2', round(d['value'],3))" >> gpurun_out/exp_outer.txt
  done
done

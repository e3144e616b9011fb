set -u
mkdir -p gpurun_out
for cfg in C4g C3 C2 C4; do
 for v in "20 96" "4 96" "1 96" "4 48" "4 24"; do
  set -- $v
  SV_DENSE_MIN_COST=$1 SV_DA_MIN_COST=$2 timeout 300 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --no-grad 2>&1 | python -c "import sys,json
for l in sys.stdin:
  if l.startswith('{'): d=json.loads(l); print('$cfg DMIN=$1 DAMIN=$2', d['value'], d['ms_per_step'])
  else: print(l.rstrip()[:200])" >> gpurun_out/exp_dense.txt
 done
done

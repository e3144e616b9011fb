set -x
mkdir -p gpurun_out
for cfg in C4g C3 C2; do
 for v in "11 1" "10 1" "10 2" "9 2" "9 3"; do
  set -- $v
  SV_DUAL_K=$1 SV_DUAL_CTAS=$2 timeout 300 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | python -c "import sys,json
for l in sys.stdin:
  if l.startswith('{'): d=json.loads(l); print('$cfg K=$1 C=$2', d['value'], d['ms_per_step'])
  else: print(l.rstrip()[:200])" >> gpurun_out/exp_dual.txt
 done
done

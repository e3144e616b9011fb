set -u
mkdir -p gpurun_out
for v in "11 3" "10 4" "10 5" "10 6" "9 8"; do
  set -- $v
  echo "== K=$1 CTAS=$2" >> gpurun_out/exp_fwd.txt
  SV_FWD_K=$1 SV_FWD_GRID_CTAS=$2 timeout 300 python tools/experiments/exp_pass_cost.py 2>&1 | grep rand11 | grep -E "depth (1|4|12):" >> gpurun_out/exp_fwd.txt
  SV_FWD_K=$1 SV_FWD_GRID_CTAS=$2 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-grad 2>&1 | python -c "import sys,json
for l in sys.stdin:
  if l.startswith('{'): d=json.loads(l); print('C4', d['value'], d['ms_per_step'])" >> gpurun_out/exp_fwd.txt
done

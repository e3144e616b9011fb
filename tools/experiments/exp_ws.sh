set -u
for v in "0 0" "3 0" "2 2"; do
  set -- $v
  echo "== SV_WS=$1 GRID_CTAS=$2" >> gpurun_out/exp_ws.txt
  env SV_WS=$1 $( [ "$2" != 0 ] && echo SV_FWD_GRID_CTAS=$2 ) EXP_DEPTHS=1,2,4,12 timeout 300 python tools/experiments/exp_pass_cost.py 2>&1 | grep rand >> gpurun_out/exp_ws.txt
  env SV_WS=$1 $( [ "$2" != 0 ] && echo SV_FWD_GRID_CTAS=$2 ) timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-grad 2>&1 | python -c "import sys,json
for l in sys.stdin:
  if l.startswith('{'): d=json.loads(l); print('C4', round(d['value'],1), d['E'])" >> gpurun_out/exp_ws.txt
done
SV_WS=3 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1 >> gpurun_out/exp_ws.txt

for v in "0 96" "0 200" "0 300" "0 150" "99 96"; do
  set -- $v
  SV_DA_MIN_QUBITS=$1 SV_DA_MIN_COST=$2 timeout 300 python bench.py --config C2 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | python -c "import sys,json
for l in sys.stdin:
  if l.startswith('{'): d=json.loads(l); print('C2 minq=$1 mincost=$2', round(d['value'],2))" >> gpurun_out/c2sweep.txt
  SV_DA_MIN_QUBITS=$1 SV_DA_MIN_COST=$2 timeout 300 python bench.py --config C4g --steps 2 --warmup 2 --no-cpu-baseline 2>&1 | python -c "import sys,json
for l in sys.stdin:
  if l.startswith('{'): d=json.loads(l); print('C4g minq=$1 mincost=$2', round(d['value'],3))" >> gpurun_out/c2sweep.txt
done

# usage: bash tools/experiments/exp_grad.sh TAG  -> appends C2/C3/C4g grad evals/s lines to gpurun_out/exp_grad.txt
set -u
mkdir -p gpurun_out
for cfg in C2 C3 C4g; do
  timeout 300 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | python -c "import sys,json
for l in sys.stdin:
  if l.startswith('{'): d=json.loads(l); print('$1 $cfg', round(d['value'],3), round(d['ms_per_step'],2))" >> gpurun_out/exp_grad.txt
done

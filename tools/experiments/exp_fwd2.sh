set -u
mkdir -p gpurun_out
for v in "11 3" "11 2" "10 3" "10 4" "10 5"; do
  set -- $v
  echo "== K=$1 CTAS=$2" >> gpurun_out/exp_fwd2.txt
  EXP_WIDTH=10 EXP_DEPTHS=8,16,32 SV_FWD_K=$1 SV_FWD_GRID_CTAS=$2 timeout 300 python tools/experiments/exp_pass_cost.py 2>&1 | grep rand >> gpurun_out/exp_fwd2.txt
done

set -u
for v in "96 2" "48 2" "200 2" "96 1" "32 2"; do
  set -- $v
  SV_DA_MIN_COST=$1 SV_DA_MAX_TILE=$2 bash tools/experiments/exp_grad.sh "da_min=$1_tile=$2"
done

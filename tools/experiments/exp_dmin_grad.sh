for v in 20 1; do
  SV_DENSE_MIN_COST=$v bash tools/experiments/exp_grad.sh "dmin=$v"
done

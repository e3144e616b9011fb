for v in 0 1; do
  SV_DA_MAX_OUTER=$v bash tools/experiments/exp_grad.sh "outer=$v"
done

for v in ${DAPP_LIST:-2 3 4}; do
  SV_DA_MAX_PER_PASS=$v bash tools/experiments/exp_grad.sh "da_per_pass=$v"
done

# builds libsv with compile-time knobs and measures the gradient configs for each
set -u
for defs in "" "-DSV_DUAL_SINGLE_BUF=1" "-DSV_DUAL_CTAS=4 -DSV_DUAL_SINGLE_BUF=1"; do
  rm -f paper_2406_17248_b200/libsv.so
  SV_NVCC_DEFS="$defs" python build.py > /dev/null 2>&1
  tag=$(echo "defs[$defs]" | tr ' ' '_')
  bash tools/experiments/exp_grad.sh "$tag"
done
rm -f paper_2406_17248_b200/libsv.so; python build.py > /dev/null 2>&1

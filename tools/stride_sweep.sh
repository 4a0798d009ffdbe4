# force / build time vs the padded row stride (build-time define), config 4 in cell order
for S in ${STRIDES:-192 160 152}; do
  NVCC_EXTRA="-DLJ_PADDED_ROW_STRIDE=$S" python -c "from paper_1806_05713_b200 import build as b; b.build(force=True)" > /dev/null
  echo "stride=$S"; python tools/order_time.py 4 2>&1 | grep '"padded": true'
done

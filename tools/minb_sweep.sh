# build liblj with different k_force min-blocks bounds and time config 4 (cell order) force steps
set -e
for MB in ${MBS:-5 1 5 1}; do
  NVCC_EXTRA="-DLJ_FORCE_MINB=$MB" python -c "from paper_1806_05713_b200 import build as b; b.build(force=True)" > /dev/null
  echo "minb=$MB"; python tools/force_sweep.py 4c 2>&1 | grep '"force"' | head -2
done

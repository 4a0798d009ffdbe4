#!/bin/bash
# builder: item rows processed in pairs (ILP) vs one by one
cd "$GRAFT_REPO_ROOT"
for v in 0 1 0 1; do
  NVCC_EXTRA=-DLJ_ITEM_ROW_PAIRS=$v python -c "from paper_1806_05713_b200 import build; build.build(force=True)" > gpurun_out/jj_build_$v.log 2>&1
  timeout 300 python tools/build_time.py 4 >> gpurun_out/jj_time_$v.log 2>&1
done
python -c "from paper_1806_05713_b200 import build; build.build(force=True)" > /dev/null 2>&1

#!/bin/bash
# predicated partner gathers (no request for lanes past their row's end): force timing A/B
cd "$GRAFT_REPO_ROOT"
for v in 0 1 2; do
  NVCC_EXTRA=-DLJ_GATHER_PRED=$v python -c "from paper_1806_05713_b200 import build; build.build(force=True)" > gpurun_out/cc_build_$v.log 2>&1
  timeout 300 python tools/build_time.py 4 > gpurun_out/cc_force_$v.log 2>&1
  timeout 300 python tools/build_time.py 3 > gpurun_out/cc_force3_$v.log 2>&1
done
python -c "from paper_1806_05713_b200 import build; build.build(force=True)" > gpurun_out/cc_build.log 2>&1

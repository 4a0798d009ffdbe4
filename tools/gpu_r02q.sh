#!/bin/bash
# v5 (warp-specialised builder) validation: list/rebuild/MD parity, build time, bench.
cd "$GRAFT_REPO_ROOT"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/q_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "rebuild or list or deferred or drifted or overflow or half_cells" > gpurun_out/q_parity.log 2>&1
echo "EXIT $?" >> gpurun_out/q_parity.log
timeout 600 python -m pytest tests/test_gpu_md.py tests/test_gpu_fullsize.py -m gpu -x -q > gpurun_out/q_md.log 2>&1
echo "EXIT $?" >> gpurun_out/q_md.log
timeout 300 python tools/build_time.py > gpurun_out/q_build_time.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/q_bench.log 2>&1
# the same timing with the v4 builder on the rebuild path
NVCC_EXTRA=-DLJ_BUILDER_V5=0 python -c "from paper_1806_05713_b200 import build; build.build(force=True)" > gpurun_out/q_build_v4.log 2>&1
timeout 300 python tools/build_time.py > gpurun_out/q_build_time_v4.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/q_bench_v4.log 2>&1

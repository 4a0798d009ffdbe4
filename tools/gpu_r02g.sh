#!/bin/bash
# round 2, call G: builder with k_cell_setup + cp.async prefetch of the next cell's setup
cd "$GRAFT_REPO_ROOT"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/g_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_md.py tests/test_gpu_fullsize.py -m gpu -q -k "list or drifted or rebuild or graph or half_cells or fullsize or nve" > gpurun_out/g_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/g_pytest.log
timeout 600 python tools/build_time.py 3,4 > gpurun_out/g_build_time.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/g_bench.log 2>&1; echo "rc=$?" >> gpurun_out/g_bench.log
ARGS="--steps 12 --warmup 3 --no-e2e --no-cpu-baseline --no-graph"
timeout 300 python bench.py $ARGS > gpurun_out/g_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_list_v4 -s 2 -c 1 -o gpurun_out/g_list python bench.py $ARGS > gpurun_out/g_ncu_list.log 2>&1; echo ncu=$? >> gpurun_out/g_plain.log

#!/bin/bash
# interleaved padded list (LJ_LIST_INTERLEAVED): parity, timing, bench A/B
cd "$GRAFT_REPO_ROOT"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "interleaved or rebuild_fused or deferred or overflowed or drifted or padded" > gpurun_out/s_parity.log 2>&1
echo "EXIT $?" >> gpurun_out/s_parity.log
timeout 300 python tools/build_time.py > gpurun_out/s_build_time.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/s_bench_il.log 2>&1
LJ_LIST_INTERLEAVE=0 timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/s_bench_plain.log 2>&1
timeout 900 python -m pytest tests/test_gpu_md.py tests/test_gpu_fullsize.py -m gpu -x -q > gpurun_out/s_md.log 2>&1
echo "EXIT $?" >> gpurun_out/s_md.log

#!/bin/bash
# interleaved list, compile-time offsets: parity + timing A/B
cd "$GRAFT_REPO_ROOT"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/t_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "interleaved or force_parity or padded or rebuild_fused" > gpurun_out/t_parity.log 2>&1
echo "EXIT $?" >> gpurun_out/t_parity.log
timeout 300 python tools/build_time.py 4 > gpurun_out/t_build_time.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/t_bench_il.log 2>&1
LJ_LIST_INTERLEAVE=0 timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/t_bench_plain.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/t_bench_il2.log 2>&1

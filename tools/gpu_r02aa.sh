#!/bin/bash
# fused rebuild + kick: MD parity (graph == eager bit for bit), bench A/B
cd "$GRAFT_REPO_ROOT"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/aa_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_md.py tests/test_gpu_parity.py -m gpu -x -q -k "graph or overflowed or rebuild" > gpurun_out/aa_md.log 2>&1
echo "EXIT $?" >> gpurun_out/aa_md.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/aa_bench_fused.log 2>&1
LJ_FUSE_FORCE=0 timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/aa_bench_plain.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/aa_bench_fused2.log 2>&1

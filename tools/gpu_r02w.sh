#!/bin/bash
# end-to-end step graph (graph_host_io): parity test + bench e2e
cd "$GRAFT_REPO_ROOT"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/w_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_md.py -m gpu -x -q > gpurun_out/w_md.log 2>&1
echo "EXIT $?" >> gpurun_out/w_md.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/w_bench.log 2>&1; echo "rc=$?" >> gpurun_out/w_bench.log

#!/bin/bash
cd "$GRAFT_REPO_ROOT"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/m_build.log 2>&1
timeout 600 python bench.py > gpurun_out/m_bench.log 2>&1; echo "rc=$?" >> gpurun_out/m_bench.log
timeout 600 python bench.py --config 3 --no-cpu-baseline > gpurun_out/m_bench_c3.log 2>&1; echo "rc=$?" >> gpurun_out/m_bench_c3.log

#!/bin/bash
cd "$GRAFT_REPO_ROOT"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/p_build.log 2>&1
timeout 300 python tools/force_counter_ab.py > gpurun_out/p_counter.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/p_bench.log 2>&1

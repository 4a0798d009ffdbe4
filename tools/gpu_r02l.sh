#!/bin/bash
cd "$GRAFT_REPO_ROOT"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/l_build.log 2>&1
timeout 600 python bench.py > gpurun_out/l_bench.log 2>&1; echo "rc=$?" >> gpurun_out/l_bench.log
( time timeout 2400 python -m pytest tests/test_gpu_checked.py -m gpu -q ) > gpurun_out/l_pytest_checked.log 2>&1; echo "rc=$?" >> gpurun_out/l_pytest_checked.log

#!/bin/bash
# round 2, call K: the bounds-checked build over the parity subset; the graph-vs-oracle MD test
cd "$GRAFT_REPO_ROOT"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/k_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_md.py -m gpu -q -k "oracle" > gpurun_out/k_pytest_md.log 2>&1; echo "rc=$?" >> gpurun_out/k_pytest_md.log
timeout 2700 python -m pytest tests/test_gpu_checked.py -m gpu -q > gpurun_out/k_pytest_checked.log 2>&1; echo "rc=$?" >> gpurun_out/k_pytest_checked.log

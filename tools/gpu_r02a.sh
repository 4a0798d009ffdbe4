#!/bin/bash
# round 2, call A: new parity tests, lanes sweep + B-15 microbenchmarks, bench line
cd "$GRAFT_REPO_ROOT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/a_smi.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_cutoff.py tests/test_gpu_parity.py -m gpu -q --maxfail=20 \
    -k "cutoff or overflow or force_parity or counterexample or deferred" > gpurun_out/a_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/a_pytest.log
timeout 600 python tools/roofline_b15.py gpurun_out/r02_b15.json > gpurun_out/a_b15.log 2>&1
echo "b15 rc=$?" >> gpurun_out/a_b15.log
timeout 600 python bench.py > gpurun_out/a_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/a_bench.log

#!/bin/bash
# round 2, call F: rowset force kernel -- parity + timing
cd "$GRAFT_REPO_ROOT"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/f_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cutoff.py -m gpu -q -k "force_parity or cutoff_edge" > gpurun_out/f_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/f_pytest.log
timeout 600 python tools/force_variants.py 4 > gpurun_out/f_variants4.log 2>&1
timeout 600 python tools/force_variants.py 3 > gpurun_out/f_variants3.log 2>&1

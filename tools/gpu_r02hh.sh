#!/bin/bash
cd "$GRAFT_REPO_ROOT"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/hh_build.log 2>&1
timeout 900 python tools/e2e_probe.py 40 > gpurun_out/hh_e2e_probe.log 2>&1
timeout 600 python -m pytest tests/test_gpu_md.py -m gpu -q -k host_io > gpurun_out/hh_md.log 2>&1; echo "EXIT $?" >> gpurun_out/hh_md.log

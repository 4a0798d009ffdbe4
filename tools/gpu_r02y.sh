#!/bin/bash
cd "$GRAFT_REPO_ROOT"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/y_build.log 2>&1
timeout 300 python tools/pcie_probe.py > gpurun_out/y_pcie.log 2>&1
timeout 600 python tools/e2e_probe.py 40 > gpurun_out/y_e2e_probe.log 2>&1

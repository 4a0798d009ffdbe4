#!/bin/bash
# B-15 microbenchmarks refreshed with the interleaved list's replays
cd "$GRAFT_REPO_ROOT"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ee_build.log 2>&1
timeout 1200 python tools/roofline_b15.py gpurun_out/ee_b15.json > gpurun_out/ee_b15.log 2>&1

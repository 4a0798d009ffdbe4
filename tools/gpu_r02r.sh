#!/bin/bash
# index-stream layout probe (row-major vs warp-tiled padded list)
cd "$GRAFT_REPO_ROOT"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r_build.log 2>&1
timeout 600 python tools/layout_probe.py 4 > gpurun_out/r_layout4.log 2>&1
timeout 300 python tools/layout_probe.py 3 > gpurun_out/r_layout3.log 2>&1

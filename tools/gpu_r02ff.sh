#!/bin/bash
cd "$GRAFT_REPO_ROOT"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ff_build.log 2>&1
timeout 600 python tools/e2e_timeline.py 30 > gpurun_out/ff_timeline.log 2>&1

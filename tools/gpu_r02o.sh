#!/bin/bash
cd "$GRAFT_REPO_ROOT"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/o_build.log 2>&1
timeout 600 python tools/force_stream_idx.py > gpurun_out/o_stream.log 2>&1; echo "rc=$?" >> gpurun_out/o_stream.log

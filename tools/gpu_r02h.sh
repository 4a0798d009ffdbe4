#!/bin/bash
cd "$GRAFT_REPO_ROOT"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/h_build.log 2>&1
timeout 300 python tools/force_g_compare.py > gpurun_out/h_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_force -s 1 -c 5 -o gpurun_out/h_force python tools/force_g_compare.py > gpurun_out/h_ncu.log 2>&1; echo ncu=$? >> gpurun_out/h_plain.log

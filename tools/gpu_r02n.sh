#!/bin/bash
# round 2, call N: final launch list + ncu captures of the force kernel and the builder (eager steps)
cd "$GRAFT_REPO_ROOT"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/n_build.log 2>&1
ARGS="--steps 12 --warmup 3 --no-e2e --no-cpu-baseline --no-graph"
timeout 300 python bench.py $ARGS > gpurun_out/n_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/n_launches.csv python bench.py $ARGS > gpurun_out/n_ncu_launches.log 2>&1; echo ncu1=$? >> gpurun_out/n_plain.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_force<" -s 5 -c 1 -o gpurun_out/n_force python bench.py $ARGS > gpurun_out/n_ncu_force.log 2>&1; echo ncu2=$? >> gpurun_out/n_plain.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_list_v4 -s 2 -c 1 -o gpurun_out/n_list python bench.py $ARGS > gpurun_out/n_ncu_list.log 2>&1; echo ncu3=$? >> gpurun_out/n_plain.log

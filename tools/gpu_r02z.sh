#!/bin/bash
# launch list of the bench's step (eager variant: ncu cannot list the kernel nodes of a graph with
# conditional nodes), interleaved list
cd "$GRAFT_REPO_ROOT"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/z_build.log 2>&1
ARGS="--steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-graph --repeats 1"
python bench.py $ARGS > gpurun_out/z_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/z_launches.csv python bench.py $ARGS > gpurun_out/z_ncu_launches.log 2>&1; echo ncu=$? >> gpurun_out/z_plain.log

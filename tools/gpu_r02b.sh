#!/bin/bash
# round 2, call B: full GPU suite (NCCL test included), smoke, bench (graph + torchrun graph_collective),
# launch list + ncu --set full of the force kernel and the builder
cd "$GRAFT_REPO_ROOT"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --maxfail=20 > gpurun_out/b_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/b_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/b_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/b_smoke.log
timeout 600 python bench.py > gpurun_out/b_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/b_bench.log
LJ_FORCE_COLLECTIVES=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
    --master-port 29511 bench.py --gpus 1 --no-cpu-baseline > gpurun_out/b_bench_torchrun.log 2>&1; echo "rc=$?" >> gpurun_out/b_bench_torchrun.log
timeout 300 python bench.py --gpus 2 > gpurun_out/b_bench_gpus2.log 2>&1; echo "rc=$? (expected: refuses, 1 GPU)" >> gpurun_out/b_bench_gpus2.log
ARGS="--steps 12 --warmup 3 --no-e2e --no-cpu-baseline --no-graph"
timeout 300 python bench.py $ARGS > gpurun_out/b_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/b_launches.csv python bench.py $ARGS > gpurun_out/b_ncu_launches.log 2>&1; echo ncu1=$? >> gpurun_out/b_plain.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_force -s 5 -c 1 -o gpurun_out/b_force python bench.py $ARGS > gpurun_out/b_ncu_force.log 2>&1; echo ncu2=$? >> gpurun_out/b_plain.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_list_v4 -s 2 -c 1 -o gpurun_out/b_list python bench.py $ARGS > gpurun_out/b_ncu_list.log 2>&1; echo ncu3=$? >> gpurun_out/b_plain.log

#!/bin/bash
# round 2, call C: the other bench lines (configs 2/3 full + half, config 5 NVE 1000 steps,
# reference arm), and the no-re-sort locality cost at P = 1 (graph vs graph_collective)
cd "$GRAFT_REPO_ROOT"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c_build.log 2>&1
for cfg in 2 3; do for lst in full half; do
  timeout 600 python bench.py --config $cfg --list $lst > gpurun_out/c_bench_c${cfg}_${lst}.log 2>&1; echo "rc=$?" >> gpurun_out/c_bench_c${cfg}_${lst}.log
done; done
timeout 1200 python bench.py --config 5 --no-e2e > gpurun_out/c_bench_c5.log 2>&1; echo "rc=$?" >> gpurun_out/c_bench_c5.log
timeout 600 python tools/unsorted_build_time.py > gpurun_out/c_unsorted.log 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/c_bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/c_bench_ref.log
LJ_FORCE_COLLECTIVES=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
    --master-port 29512 bench.py --gpus 1 --no-cpu-baseline --no-e2e > gpurun_out/c_bench_torchrun_graph.log 2>&1; echo "rc=$?" >> gpurun_out/c_bench_torchrun_graph.log
LJ_FORCE_COLLECTIVES=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
    --master-port 29513 bench.py --gpus 1 --no-cpu-baseline --no-e2e --no-graph > gpurun_out/c_bench_torchrun_eager.log 2>&1; echo "rc=$?" >> gpurun_out/c_bench_torchrun_eager.log

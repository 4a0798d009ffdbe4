#!/bin/bash
# round 2, call E: graph_collective with the NVLink-sourced re-sort
cd "$GRAFT_REPO_ROOT"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/e_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_nccl.py tests/test_gpu_push.py tests/test_gpu_md.py -m gpu -q > gpurun_out/e_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/e_pytest.log
LJ_FORCE_COLLECTIVES=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
    --master-port 29512 bench.py --gpus 1 --no-cpu-baseline --no-e2e > gpurun_out/e_bench_torchrun_graph.log 2>&1; echo "rc=$?" >> gpurun_out/e_bench_torchrun_graph.log

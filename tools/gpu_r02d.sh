#!/bin/bash
# round 2, call D: drifted-storage builder (rank path), graph_collective bench, interleaved-index experiment
cd "$GRAFT_REPO_ROOT"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/d_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "list or drifted" > gpurun_out/d_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/d_pytest.log
timeout 600 python tools/unsorted_build_time.py > gpurun_out/d_unsorted.log 2>&1
LJ_FORCE_COLLECTIVES=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
    --master-port 29512 bench.py --gpus 1 --no-cpu-baseline --no-e2e > gpurun_out/d_bench_torchrun_graph.log 2>&1; echo "rc=$?" >> gpurun_out/d_bench_torchrun_graph.log
timeout 600 python tools/interleave_probe.py > gpurun_out/d_interleave.log 2>&1; echo "rc=$?" >> gpurun_out/d_interleave.log
timeout 600 python bench.py --config 2 --list full --no-cpu-baseline --no-e2e > gpurun_out/d_bench_c2.log 2>&1

#!/bin/bash
# round 2, call I: full validation (GPU suite, smoke) + bench lines after the builder and graph changes
cd "$GRAFT_REPO_ROOT"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/i_build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q --maxfail=30 > gpurun_out/i_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/i_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/i_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/i_smoke.log
timeout 600 python bench.py > gpurun_out/i_bench.log 2>&1; echo "rc=$?" >> gpurun_out/i_bench.log
LJ_FORCE_COLLECTIVES=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
    --master-port 29512 bench.py --gpus 1 --no-cpu-baseline --no-e2e > gpurun_out/i_bench_torchrun_graph.log 2>&1; echo "rc=$?" >> gpurun_out/i_bench_torchrun_graph.log
timeout 1200 python bench.py --config 5 --no-e2e > gpurun_out/i_bench_c5.log 2>&1; echo "rc=$?" >> gpurun_out/i_bench_c5.log

#!/bin/bash
# round 2, call BB: final validation (interleaved list, e2e graph) (GPU suite, smoke, bench lines)
cd "$GRAFT_REPO_ROOT"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/bb_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q --maxfail=30 > gpurun_out/bb_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/bb_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/bb_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/bb_smoke.log
timeout 900 python bench.py > gpurun_out/bb_bench.log 2>&1; echo "rc=$?" >> gpurun_out/bb_bench.log
LJ_FORCE_COLLECTIVES=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
    --master-port 29512 bench.py --gpus 1 --no-cpu-baseline --no-e2e > gpurun_out/bb_bench_torchrun_graph.log 2>&1; echo "rc=$?" >> gpurun_out/bb_bench_torchrun_graph.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bb_bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/bb_bench_ref.log
for c in 2 3; do for h in full half; do
  timeout 300 python bench.py --config $c --list $h --no-cpu-baseline --no-e2e > gpurun_out/bb_bench_c${c}_$h.log 2>&1
done; done
timeout 1500 python bench.py --config 5 --no-e2e > gpurun_out/bb_bench_c5.log 2>&1; echo "rc=$?" >> gpurun_out/bb_bench_c5.log

# full GPU check: tests, smoke, bench (plain and via torchrun/NCCL at P=1 with collectives forced), profiles
set -x
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?
python tools/exercise_kernels.py > gpurun_out/exercise.log 2>&1; echo exercise=$?; tail -1 gpurun_out/exercise.log
LJ_FORCE_COLLECTIVES=1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 20 --warmup 5 --no-e2e > gpurun_out/bench_torchrun.log 2>&1; echo torchrun=$?
python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo ref=$?
# ncu does not list the kernel nodes of a graph with conditional nodes: the launch list and
# the captures use the eager step (--no-graph), same kernels
ARGS="--steps 12 --warmup 3 --no-e2e --no-cpu-baseline --no-graph"
python bench.py $ARGS > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/launches.csv python bench.py $ARGS > gpurun_out/ncu_launches.log 2>&1; echo ncu1=$?
ncu --set full --clock-control none --import-source on -k regex:k_force -s 5 -c 1 -o gpurun_out/force_prof python bench.py $ARGS > gpurun_out/ncu_force.log 2>&1; echo ncu2=$?
ncu --set full --clock-control none --import-source on -k regex:k_list_v4 -s 2 -c 1 -o gpurun_out/list_prof python bench.py $ARGS > gpurun_out/ncu_list.log 2>&1; echo ncu3=$?

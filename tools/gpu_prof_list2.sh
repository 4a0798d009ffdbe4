ARGS="--steps 12 --warmup 3 --no-e2e --no-cpu-baseline"
python bench.py $ARGS > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_list_v2 -s 1 -c 1 -o gpurun_out/list_v3 python bench.py $ARGS > gpurun_out/ncu_list.log 2>&1; echo ncu=$?

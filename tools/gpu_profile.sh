# bench + launch list + ncu --set full of the force and list kernels (one GPU)
ARGS="--steps 20 --warmup 5 --no-e2e --no-cpu-baseline"
python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?
python bench.py $ARGS > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file gpurun_out/launches.csv python bench.py $ARGS > gpurun_out/ncu_launches.log 2>&1; echo ncu1=$?
ncu --set full --clock-control none --import-source on -k regex:k_force -s 10 -c 1 -o gpurun_out/force_full python bench.py $ARGS > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
ncu --set full --clock-control none --import-source on -k regex:k_list_v4 -s 2 -c 1 -o gpurun_out/list_full python bench.py $ARGS > gpurun_out/ncu_list.log 2>&1; echo ncu3=$?

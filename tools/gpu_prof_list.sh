ARGS="--steps 12 --warmup 3 --no-e2e --no-cpu-baseline"
python bench.py $ARGS > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/launches.csv python bench.py $ARGS > gpurun_out/ncu_launches.log 2>&1; echo ncu1=$?
ncu --set full --clock-control none --import-source on -k regex:k_list_v2 -s 1 -c 1 -o gpurun_out/list_v2 python bench.py $ARGS > gpurun_out/ncu_list.log 2>&1; echo ncu2=$?
ncu --set full --clock-control none --import-source on -k regex:k_force -s 5 -c 1 -o gpurun_out/force_u4 python bench.py $ARGS > gpurun_out/ncu_force.log 2>&1; echo ncu3=$?

mkdir -p gpurun_out
CMD="python bench.py --steps 5 --warmup 3 --cpu-seconds 3"
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/clocks_r1c.csv &
SMI=$!
$CMD > gpurun_out/plain_r1c.log 2>&1
kill $SMI
$CMD > gpurun_out/plain_r1c_2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k1_|k2_|k0_|k1s_|k_stats|kc_" -c 3000 --csv --log-file gpurun_out/launches_r1c.csv $CMD > gpurun_out/ncu_launch_r1c.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k1_accumulate_many -c 1 -o gpurun_out/kmany_r1c -f $CMD > gpurun_out/ncu_kmany.log 2>&1
ls gpurun_out | grep r1c

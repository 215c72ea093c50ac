mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_b.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k1_|k2_|k0_|k1s_|k_stats" --csv --log-file gpurun_out/launches_r1b.csv $CMD > gpurun_out/ncu_launch_b.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k2_adam -s 2 -c 1 -o gpurun_out/k2_r1b -f $CMD > gpurun_out/ncu_k2b.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k1_accumulate -s 20 -c 1 -o gpurun_out/k1_r1b -f $CMD > gpurun_out/ncu_k1b.log 2>&1
CMD2="python bench.py --config base --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD2 > gpurun_out/plain_base.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k1_|k2_|k0_|k1s_" --csv --log-file gpurun_out/launches_base_r1b.csv $CMD2 > gpurun_out/ncu_launch_base.log 2>&1
ls gpurun_out

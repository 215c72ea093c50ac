set -x
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k1_|k2_|k0_|k1s_" --csv --log-file gpurun_out/launches_r1.csv $CMD > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k2_adam -s 2 -c 1 -o gpurun_out/k2_r1 -f $CMD > gpurun_out/ncu_k2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k1_accumulate -s 20 -c 1 -o gpurun_out/k1_r1 -f $CMD > gpurun_out/ncu_k1.log 2>&1
ls -la gpurun_out

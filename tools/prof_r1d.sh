# round-1 final profile of the default N=1 bench (fused last micro-batch): launch list + one full capture each of
# the two dominant kernels (k1_accumulate_1 add, k12_fused) and of k12_fused at c = 1 (base)
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_d.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k1_|k2_|k0_|k1s_|k12_|kc_" --csv --log-file gpurun_out/launches_r1d.csv $CMD > gpurun_out/ncu_launch_d.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k12_fused -s 2 -c 1 -o gpurun_out/k12_r1d -f $CMD > gpurun_out/ncu_k12d.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k1_accumulate -s 20 -c 1 -o gpurun_out/k1_r1d -f $CMD > gpurun_out/ncu_k1d.log 2>&1
CMD2="python bench.py --config base --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD2 > gpurun_out/plain_base_d.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k12_fused -s 2 -c 1 -o gpurun_out/k12base_r1d -f $CMD2 > gpurun_out/ncu_k12based.log 2>&1
ls gpurun_out | grep r1d

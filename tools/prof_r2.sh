# round-2 profile of the default N = 1 bench (the headline: fuse_final = 0, K1 passes + K0 + K2): launch list of
# the library's kernels + one `ncu --set full` capture each of the two dominant kernels (k1_accumulate_1 add,
# k2_adam_1), and the whole -m gpu suite with per-test durations.
set -x
O=gpurun_out/r2k
mkdir -p $O
cat .head_sha > $O/head.txt
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 python bench.py > $O/bench_n1.json 2> $O/bench_n1.err
$CMD > $O/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k1_|k2_|k0_|k1s_|k12_|kc_" --csv --log-file $O/launches_r2.csv $CMD > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_accumulate -s 20 -c 1 -o $O/k1_r2 -f $CMD > $O/ncu_k1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k2_adam -s 2 -c 1 -o $O/k2_r2 -f $CMD > $O/ncu_k2.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rs --durations=40 > $O/gpu_tests.log 2>&1; echo "pytest rc=$?" >> $O/gpu_tests.log
echo done

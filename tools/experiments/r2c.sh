#!/bin/bash
# round 2, single GPU: C3 at W=8 over virtual ranks, the W=1 bench headline, the real-producer train mode,
# straggler calibration on the real model, oracle per-config timings, launch list of the bench.
set -x
O=gpurun_out/r2c
mkdir -p $O
git_sha=$(cat .git_sha 2>/dev/null)
nvidia-smi -L
python -m pytest tests/test_gpu_virtual.py -k c3 -q -s -x > $O/c3_virtual_w8.log 2>&1
python bench.py > $O/bench_n1.json 2> $O/bench_n1.err
python bench.py --mode train --steps 4 --warmup 2 > $O/train_n1_c16.json 2> $O/train_n1_c16.err
python bench.py --mode train --update-freq 1 --steps 10 --warmup 3 > $O/train_n1_c1.json 2> $O/train_n1_c1.err
python tools/straggler_calibrate.py --measure 240 --out $O/straggler_measured.txt > $O/straggler.log 2>&1
python bench.py --generator real_sparse --no-e2e --no-cpu-baseline > $O/bench_sparse.json 2> $O/bench_sparse.err
timeout 900 python tools/oracle_timings.py --out $O/oracle_timings.txt > $O/oracle_timings.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu_launch.log 2>&1
echo done

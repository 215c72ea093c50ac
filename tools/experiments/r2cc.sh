#!/bin/bash
# round 2, W = 4: a longer real-peer fuzz campaign (50 cases at W = 4, 40 at W = 2, fresh seeds) and the N = 4 bench
# line with the standalone all-reduce.
set -x
O=gpurun_out/r2cc
mkdir -p $O
cat .head_sha > $O/head.txt
SMPU_FUZZ_EXAMPLES=50 SMPU_FUZZ_SEED=902 timeout 2400 python -m pytest tests/test_gpu_multi.py -v -s -k "random_cases and 4" > $O/mp_fuzz_w4.log 2>&1
SMPU_FUZZ_EXAMPLES=40 SMPU_FUZZ_SEED=903 timeout 1800 python -m pytest tests/test_gpu_multi.py -v -s -k "random_cases and 2" > $O/mp_fuzz_w2.log 2>&1
timeout 600 python bench.py --gpus 4 --no-e2e > $O/bench_n4.json 2> $O/bench_n4.err
echo done

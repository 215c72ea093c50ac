#!/bin/bash
# round 2, W = 2: the bench line with the standalone all-reduce figure; a longer real-peer fuzz campaign.
set -x
O=gpurun_out/r2bb
mkdir -p $O
cat .head_sha > $O/head.txt
timeout 600 python bench.py --gpus 2 --no-e2e > $O/bench_n2.json 2> $O/bench_n2.err
SMPU_FUZZ_EXAMPLES=80 SMPU_FUZZ_SEED=901 timeout 2400 python -m pytest tests/test_gpu_multi.py -v -s -k "random_cases and 2" > $O/mp_fuzz.log 2>&1
echo done

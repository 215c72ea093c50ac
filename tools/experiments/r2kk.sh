#!/bin/bash
# round 2, final: one more real-peer fuzz campaign at W = 2 (60 cases, seed 904) at HEAD.
set -x
O=gpurun_out/r2kk
mkdir -p $O
cat .head_sha > $O/head.txt
SMPU_FUZZ_EXAMPLES=60 SMPU_FUZZ_SEED=904 timeout 900 python -m pytest tests/test_gpu_multi.py -v -s -k "random_cases and 2" > $O/mp_fuzz.log 2>&1
echo done

#!/bin/bash
# round 2, 1 GPU: long fuzz campaigns with fresh seeds (W = 1: 1,500 cases; W > 1 over virtual ranks: 3,000 cases).
set -x
O=gpurun_out/r2z
mkdir -p $O
cat .head_sha > $O/head.txt
SMPU_FUZZ_SEED=777 SMPU_FUZZ_EXAMPLES=3000 timeout 1800 python -m pytest tests/test_gpu_virtual_fuzz.py -q -s > $O/vfuzz.log 2>&1
SMPU_FUZZ_SEED=778 SMPU_FUZZ_EXAMPLES=1500 timeout 1800 python -m pytest tests/test_gpu_fuzz.py -q -s > $O/fuzz.log 2>&1
echo done

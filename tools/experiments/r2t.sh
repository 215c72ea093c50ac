#!/bin/bash
# round 2, 1 GPU: the W > 1 hypothesis fuzz over virtual ranks and the fp32-accumulator cases at W > 1.
set -x
O=gpurun_out/r2t
mkdir -p $O
git_head=$(cat .head_sha); echo $git_head > $O/head.txt
timeout 1500 python -m pytest tests/test_gpu_virtual_fuzz.py tests/test_gpu_virtual.py -v -s -k "fuzz or accum_fp32" > $O/virtual.log 2>&1
echo done

#!/bin/bash
# round 2, W = 2, final: the whole multi-GPU suite at HEAD (two Adam streams).
set -x
O=gpurun_out/r2ff
mkdir -p $O
cat .head_sha > $O/head.txt
timeout 1500 python -m pytest tests/test_gpu_multi.py -v > $O/multi_w2.log 2>&1
echo done

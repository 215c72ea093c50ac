#!/bin/bash
# round 2, 1 GPU: the packed-lane max fix of the K1 statistic -- the probe, the head/tail regression test, the W > 1
# fuzz, and the whole virtual-rank file.
set -x
O=gpurun_out/r2w
mkdir -p $O
cat .head_sha > $O/head.txt
./tools/k1_stats_probe > $O/probe.log 2>&1
timeout 2400 python -m pytest tests/test_gpu_virtual_fuzz.py tests/test_gpu_virtual.py -v -s > $O/virtual.log 2>&1
echo done

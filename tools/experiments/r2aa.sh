#!/bin/bash
# round 2, W = 4: random cases on real peers (tests/mp_fuzz_worker.py) at W = 2 and 4.
set -x
O=gpurun_out/r2aa
mkdir -p $O
cat .head_sha > $O/head.txt
timeout 1500 python -m pytest tests/test_gpu_multi.py -v -s -k random_cases > $O/multi_fuzz.log 2>&1
echo done

#!/bin/bash
# round 2, 1 GPU, at HEAD: configs[1] (Transformer-base, c = 1) and the configs[3] shape (Transformer-big En-Fr,
# c = 16) bench lines at N = 1.
set -x
O=gpurun_out/r2hh
mkdir -p $O
cat .head_sha > $O/head.txt
timeout 600 python bench.py --config base --no-cpu-baseline > $O/bench_base.json 2> $O/bench_base.err
timeout 600 python bench.py --config big_enfr --no-cpu-baseline --no-e2e > $O/bench_enfr.json 2> $O/bench_enfr.err
echo done

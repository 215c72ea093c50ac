#!/bin/bash
# round 2, W = 2, final: the N = 2 bench line at HEAD and the real-backward train mode at c = 1.
set -x
O=gpurun_out/r2ii
mkdir -p $O
cat .head_sha > $O/head.txt
timeout 600 python bench.py --gpus 2 > $O/bench_n2.json 2> $O/bench_n2.err
timeout 600 python bench.py --gpus 2 --mode train --update-freq 1 --steps 30 --warmup 5 > $O/train_c1.json 2> $O/train_c1.err
echo done

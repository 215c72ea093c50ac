#!/bin/bash
# round 2, W = 2: the grid flag barrier with one system fence per CTA (not per thread) -- pieces sweep + the W = 2
# parity cases of the fused all-reduce.
set -x
O=gpurun_out/r2m
mkdir -p $O
cat .head_sha > $O/head.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29641 \
  tools/c4_sweep.py --c 16,1 --mib 150 --pieces 1,2,4,8 --out $O/c4_w2_pieces.jsonl > $O/c4_w2_pieces.log 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py -v -k "world2 and fused or sharded" > $O/multi.log 2>&1
echo done

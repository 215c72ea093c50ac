#!/bin/bash
# round 2, W = 4: the all-reduce's launch shape in situ now that the all-reduce chain is the update's critical path
# (r2n timelines): CTAs x threads x unroll, with ar_pieces 1 / 2, at c = 16 and 1.
set -x
O=gpurun_out/r2o
mkdir -p $O
cat .head_sha > $O/head.txt
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29651 \
  tools/c4_sweep.py --c 16,1 --mib 150 --pieces 1,2 --shape 148x256x1,148x256x2,296x256x1,148x512x1,296x256x2,74x512x2 \
  --out $O/c4_w4_shape.jsonl > $O/c4_w4_shape.log 2>&1
echo done

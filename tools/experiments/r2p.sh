#!/bin/bash
# round 2, W = 4 then W = 2: fewer, wider all-reduce CTAs (r2o: 74 x 512 x 2 reaches 611 GB/s in situ at the
# default's step time) -- shape sweep around it, and the SM all-reduce with that footprint beside a real backward.
set -x
O=gpurun_out/r2p
mkdir -p $O
cat .head_sha > $O/head.txt
SH=148x256x1,74x512x2,48x512x2,96x512x2,74x256x2,37x512x2
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29661 \
  tools/c4_sweep.py --c 16,1 --mib 150 --pieces 2 --shape $SH --out $O/c4_w4_shape.jsonl > $O/c4_w4_shape.log 2>&1
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29662 \
  tools/c4_sweep.py --c 16,1 --mib 150 --pieces 2 --shape $SH --out $O/c4_w2_shape.jsonl > $O/c4_w2_shape.log 2>&1
timeout 600 python bench.py --gpus 4 --mode train --update-freq 1 --steps 30 --warmup 5 --ar-copy-engine 0 --ar-ctas 74 --ar-threads 512 --ar-unroll 2 > $O/train_c1_sm74.json 2> $O/train_c1_sm74.err
timeout 600 python bench.py --gpus 4 --mode train --update-freq 1 --steps 30 --warmup 5 --ar-copy-engine 0 --ar-ctas 37 --ar-threads 512 --ar-unroll 2 > $O/train_c1_sm37.json 2> $O/train_c1_sm37.err
timeout 600 python bench.py --gpus 4 --mode train --update-freq 1 --steps 30 --warmup 5 --ar-copy-engine 1 > $O/train_c1_ce1.json 2> $O/train_c1_ce1.err
echo done

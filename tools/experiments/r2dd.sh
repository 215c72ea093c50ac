#!/bin/bash
# round 2, W = 4: two Adam streams (pieces alternate) -- C4 pieces sweep at c = 16 / 1, N = 2 / 4 bench, the fused
# multi-GPU parity subset, the virtual suite.
set -x
O=gpurun_out/r2dd
mkdir -p $O
cat .head_sha > $O/head.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29671 \
  tools/c4_sweep.py --c 16,1 --mib 150 --pieces 1,2,4 --out $O/c4_w4.jsonl > $O/c4_w4.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29672 \
  tools/c4_sweep.py --c 16,1 --mib 150 --pieces 1,2,4 --out $O/c4_w2.jsonl > $O/c4_w2.log 2>&1
timeout 600 python bench.py --gpus 4 --no-e2e > $O/bench_n4.json 2> $O/bench_n4.err
timeout 900 python -m pytest tests/test_gpu_virtual.py -q -x > $O/virtual.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_multi.py -q -x -k "fused or sharded or copy_engine or random" > $O/multi.log 2>&1
echo done

#!/bin/bash
# round 2, W = 2: ar_copy_engine 3 (every piece split between the SM kernel and the copy engines) -- parity on
# virtual ranks and real peers, and the C4 comparison against the SM kernel alone at c = 16 / 1.
set -x
O=gpurun_out/r2gg
mkdir -p $O
cat .head_sha > $O/head.txt
timeout 600 python -m pytest tests/test_gpu_virtual.py tests/test_gpu_virtual_fuzz.py -q -x -k "copy_engine or fuzz" > $O/virtual.log 2>&1
timeout 600 python -m pytest tests/test_gpu_multi.py -q -x -k "copy_engine and 2-True-3" > $O/multi.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29681 \
  tools/c4_sweep.py --c 16,1 --mib 150 --pieces 2 --ce 0,3 --out $O/c4_w2.jsonl > $O/c4_w2.log 2>&1
echo done

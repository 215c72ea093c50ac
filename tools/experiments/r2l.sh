#!/bin/bash
# round 2, W = 4 (gpurun --gpus 4): the bucket kernels' grid flag barrier -- the whole multi-GPU suite, the pieces
# sweep at W = 2 / 4 (per-launch overhead), the N = 2 / 4 bench lines, the rotating-partner CE probe.
set -x
O=gpurun_out/r2l
mkdir -p $O
cat .head_sha > $O/head.txt
timeout 1500 python -m pytest tests/test_gpu_multi.py -v > $O/multi_w4.log 2>&1
timeout 600 python -m pytest tests/test_gpu_virtual.py -q -k "world_bitwise or pieces or copy_engine" > $O/virtual.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29631 \
  tools/c4_sweep.py --c 16,1 --mib 150 --pieces 1,2,4,8 --out $O/c4_w4_pieces.jsonl > $O/c4_w4_pieces.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29632 \
  tools/c4_sweep.py --c 16,1 --mib 150 --pieces 1,2,4,8 --out $O/c4_w2_pieces.jsonl > $O/c4_w2_pieces.log 2>&1
timeout 600 python bench.py --gpus 4 --no-e2e > $O/bench_n4.json 2> $O/bench_n4.err
timeout 600 python bench.py --gpus 2 --no-e2e > $O/bench_n2.json 2> $O/bench_n2.err
timeout 300 python tools/ce_probe.py 256 > $O/ce_probe.jsonl 2> $O/ce_probe.err
echo done

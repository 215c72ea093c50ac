#!/bin/bash
# round 2, final: the driver's own N > 1 launch (torchrun) of the default bench at N = 4, and its reference arm.
set -x
O=gpurun_out/r2jj
mkdir -p $O
cat .head_sha > $O/head.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29691 \
  bench.py --gpus 4 --steps 20 --warmup 5 > $O/bench_n4_torchrun.json 2> $O/bench_n4_torchrun.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29692 \
  bench.py --impl reference --gpus 4 --steps 3 --warmup 1 > $O/ref_n4_torchrun.json 2> $O/ref_n4_torchrun.err
echo done

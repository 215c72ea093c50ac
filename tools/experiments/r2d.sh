#!/bin/bash
# round 2, W = 2 (gpurun --gpus 2): the bench self-launched without torchrun, the C4 sweep at c = 16 and 1 with the
# pipelined tail, M2 and the real-producer train mode at c = 1 (overlap vs no overlap) and c = 16.
set -x
O=gpurun_out/r2d
mkdir -p $O
nvidia-smi -L
python bench.py --gpus 2 > $O/bench_n2.json 2> $O/bench_n2.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29601 \
  tools/c4_sweep.py --c 16,1 --out $O/c4_w2.jsonl > $O/c4_w2.log 2>&1
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29602 \
  tools/c4_sweep.py --c 16,1 --mib 150 --tail-split 1,2,4,8 --out $O/c4_w2_split.jsonl > $O/c4_w2_split.log 2>&1
python bench.py --gpus 2 --mode m2 --update-freq 1 --steps 10 --warmup 3 > $O/m2_big_c1.json 2> $O/m2_big_c1.err
python bench.py --gpus 2 --mode m2 --config base --steps 10 --warmup 3 > $O/m2_base_c1.json 2> $O/m2_base_c1.err
python bench.py --gpus 2 --mode train --update-freq 1 --steps 10 --warmup 3 > $O/train_c1.json 2> $O/train_c1.err
python bench.py --gpus 2 --mode train --steps 4 --warmup 2 > $O/train_c16.json 2> $O/train_c16.err
echo done

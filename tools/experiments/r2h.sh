#!/bin/bash
# round 2 (re-entry), W = 2 (gpurun --gpus 2): the whole multi-GPU suite at HEAD, the self-launched bench at N = 2
# (replicated headline + sharded beside), the graphed real producer at c = 1 / 16 with and without overlap, the C4
# sweep at c = 16 / 1 with ar_pieces.
set -x
O=gpurun_out/r2h
mkdir -p $O
cat .head_sha > $O/head.txt
nvidia-smi topo -m > $O/topo.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_multi.py -v > $O/multi_w2.log 2>&1; echo "rc=$?" >> $O/multi_w2.log
timeout 600 python bench.py --gpus 2 > $O/bench_n2.json 2> $O/bench_n2.err
timeout 600 python bench.py --gpus 2 --mode train --update-freq 1 --steps 20 --warmup 3 > $O/train_c1.json 2> $O/train_c1.err
timeout 600 python bench.py --gpus 2 --mode train --steps 4 --warmup 2 > $O/train_c16.json 2> $O/train_c16.err
timeout 600 python bench.py --gpus 2 --mode m2 --update-freq 1 --steps 10 --warmup 3 > $O/m2_big_c1.json 2> $O/m2_big_c1.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29613 \
  tools/c4_sweep.py --c 16,1 --mib 64,150 --pieces 1,2,4,8 --out $O/c4_w2_pieces.jsonl > $O/c4_w2_pieces.log 2>&1
echo done

#!/bin/bash
# round 2, W = 4 (gpurun --gpus 4): the multi-GPU suite at W = 4 (24 + mismatch), the bench at N = 4 (headline
# replicated + sharded beside), the C4 sweep at c = 16 / 1 with ar_pieces, M2 and the graphed real producer at
# c = 1 / 16, overlap vs no overlap.
set -x
O=gpurun_out/r2f
mkdir -p $O
cat .head_sha > $O/head.txt
nvidia-smi topo -m > $O/topo.txt 2>&1
python -m pytest tests/test_gpu_virtual.py -q -k "pieces or world_bitwise" > $O/virtual_pieces.log 2>&1
python -m pytest tests/test_gpu_multi.py -v > $O/multi_w4.log 2>&1
python bench.py --gpus 4 > $O/bench_n4.json 2> $O/bench_n4.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29611 \
  tools/c4_sweep.py --c 16,1 --out $O/c4_w4.jsonl > $O/c4_w4.log 2>&1
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29612 \
  tools/c4_sweep.py --c 16,1 --mib 64,150 --pieces 1,2,4,8 --out $O/c4_w4_pieces.jsonl > $O/c4_w4_pieces.log 2>&1
python bench.py --gpus 4 --mode m2 --update-freq 1 --steps 10 --warmup 3 > $O/m2_big_c1.json 2> $O/m2_big_c1.err
python bench.py --gpus 4 --mode m2 --config base --steps 10 --warmup 3 > $O/m2_base_c1.json 2> $O/m2_base_c1.err
python bench.py --gpus 4 --mode train --update-freq 1 --steps 20 --warmup 3 > $O/train_c1.json 2> $O/train_c1.err
python bench.py --gpus 4 --mode train --steps 4 --warmup 2 > $O/train_c16.json 2> $O/train_c16.err
echo done

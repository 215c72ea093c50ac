#!/bin/bash
# round 2, W = 2 (gpurun --gpus 2): copy-engine all-reduce (smpu_config.ar_copy_engine) -- CE peer bandwidth probe,
# virtual-rank + real-peer parity, C4 sweep CE vs SM at c = 16 / 1, the graphed real producer at c = 1 with CE.
set -x
O=gpurun_out/r2i
mkdir -p $O
cat .head_sha > $O/head.txt
timeout 300 python tools/ce_probe.py 256 > $O/ce_probe.jsonl 2> $O/ce_probe.err
timeout 900 python -m pytest tests/test_gpu_virtual.py -q -k copy_engine > $O/virtual_ce.log 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py -v -k copy_engine > $O/multi_ce.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29621 \
  tools/c4_sweep.py --c 16,1 --mib 64,150 --ce 0,1 --out $O/c4_w2_ce.jsonl > $O/c4_w2_ce.log 2>&1
timeout 600 python bench.py --gpus 2 --ar-copy-engine 1 > $O/bench_n2_ce.json 2> $O/bench_n2_ce.err
timeout 600 python bench.py --gpus 2 --mode train --update-freq 1 --steps 20 --warmup 3 --ar-copy-engine 1 > $O/train_c1_ce.json 2> $O/train_c1_ce.err
timeout 600 python bench.py --gpus 2 --mode train --update-freq 1 --steps 20 --warmup 3 > $O/train_c1_sm.json 2> $O/train_c1_sm.err
echo done

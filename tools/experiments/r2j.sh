#!/bin/bash
# round 2, W = $1 (gpurun --gpus $1): the copy-engine all-reduce modes (ar_copy_engine 0 / 1 / 2) where a backward
# runs beside the exchange -- the graphed real Transformer-big producer and the M2 GEMM-load emulator at c = 1 and
# c = 16 -- plus the CE parity tests and the M1 headline with ar_pieces 2.
W=${1:-2}
set -x
O=gpurun_out/r2j_w$W
mkdir -p $O
cat .head_sha > $O/head.txt
timeout 300 ./tools/nvlink_probe 512 > $O/nvlink_probe.jsonl 2> $O/nvlink_probe.err
timeout 300 python tools/ce_probe.py 256 > $O/ce_probe.jsonl 2> $O/ce_probe.err
timeout 900 python -m pytest tests/test_gpu_virtual.py -q -k copy_engine > $O/virtual_ce.log 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py -v -k copy_engine > $O/multi_ce.log 2>&1
for ce in 0 1 2; do
  timeout 600 python bench.py --gpus $W --mode train --update-freq 1 --steps 30 --warmup 5 --ar-copy-engine $ce > $O/train_c1_ce$ce.json 2> $O/train_c1_ce$ce.err
  timeout 600 python bench.py --gpus $W --mode m2 --update-freq 1 --steps 10 --warmup 3 --ar-copy-engine $ce > $O/m2_c1_ce$ce.json 2> $O/m2_c1_ce$ce.err
done
timeout 600 python bench.py --gpus $W --mode train --steps 4 --warmup 2 --ar-copy-engine 2 > $O/train_c16_ce2.json 2> $O/train_c16_ce2.err
timeout 600 python bench.py --gpus $W --ar-pieces 2 --no-cpu-baseline > $O/bench_pieces2.json 2> $O/bench_pieces2.err
echo done

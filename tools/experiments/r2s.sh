#!/bin/bash
# round 2, W = 4 at HEAD: the whole multi-GPU suite, smoke(), the default N = 2 / 4 bench lines, the real-backward
# train mode at c = 1 / 16 (copy-engine all-reduce, the bench default there), M2 at c = 1.
set -x
O=gpurun_out/r2s
mkdir -p $O
cat .head_sha > $O/head.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 1800 python -m pytest tests/test_gpu_multi.py -v > $O/multi_w4.log 2>&1
timeout 600 python bench.py --gpus 4 > $O/bench_n4.json 2> $O/bench_n4.err
timeout 600 python bench.py --gpus 2 > $O/bench_n2.json 2> $O/bench_n2.err
timeout 600 python bench.py --gpus 4 --mode train --update-freq 1 --steps 30 --warmup 5 > $O/train_c1.json 2> $O/train_c1.err
timeout 600 python bench.py --gpus 4 --mode train --steps 4 --warmup 2 > $O/train_c16.json 2> $O/train_c16.err
timeout 600 python bench.py --gpus 4 --mode m2 --update-freq 1 --steps 10 --warmup 3 > $O/m2_c1.json 2> $O/m2_c1.err
echo done

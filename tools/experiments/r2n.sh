#!/bin/bash
# round 2, W = 4: per-stream launch timelines of the library-only update (call path) with ar_pieces 1 and 2.
set -x
O=gpurun_out/r2n
mkdir -p $O
cat .head_sha > $O/head.txt
for p in 1 2; do
  timeout 600 python bench.py --gpus 4 --steps 3 --warmup 3 --no-e2e --no-graph --ar-pieces $p --trace $O/trace_p$p.jsonl > $O/bench_p$p.json 2> $O/bench_p$p.err
done
echo done

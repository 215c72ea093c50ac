#!/bin/bash
# round 2, W = 2: degenerate buckets (one per tensor, down to 7 elements) over SM / CE all-reduces on virtual ranks;
# mismatched ar_copy_engine / ar_pieces refused on every rank; the shortened W = 8 C3 test.
set -x
O=gpurun_out/r2q
mkdir -p $O
cat .head_sha > $O/head.txt
timeout 900 python -m pytest tests/test_gpu_virtual.py -v -k "one_bucket or copy_engine or c3" > $O/virtual.log 2>&1
timeout 600 python -m pytest tests/test_gpu_multi.py -v -k "mismatch" > $O/multi.log 2>&1
echo done

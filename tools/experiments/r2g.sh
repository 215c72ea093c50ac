#!/bin/bash
# round 2 (re-entry), 1 GPU: the whole -m gpu suite at HEAD (virtual ranks included), the default N = 1 bench,
# smoke(), and the ncu launch list of the default bench.
set -x
O=gpurun_out/r2g
mkdir -p $O
git_sha=$(cat .head_sha 2>/dev/null); echo "head $git_sha" > $O/head.txt
nvidia-smi -L > $O/gpus.txt
timeout 1500 python -m pytest tests -m gpu -q -rs > $O/gpu_tests.log 2>&1; echo "pytest rc=$?" >> $O/gpu_tests.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 600 python bench.py > $O/bench_n1.json 2> $O/bench_n1.err
timeout 600 python bench.py --impl reference > $O/ref_n1.json 2> $O/ref_n1.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 3 > $O/ncu.log 2>&1
echo done

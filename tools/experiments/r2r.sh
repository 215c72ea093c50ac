#!/bin/bash
# round 2, 1 GPU, at HEAD: the whole -m gpu suite (durations), smoke(), the default N = 1 bench and the reference arm.
set -x
O=${OUT:-gpurun_out/r2r}
mkdir -p $O
cat .head_sha > $O/head.txt
timeout 2400 python -m pytest tests -m gpu -q -rs --durations=15 > $O/gpu_tests.log 2>&1; echo "pytest rc=$?" >> $O/gpu_tests.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 600 python bench.py > $O/bench_n1.json 2> $O/bench_n1.err
timeout 600 python bench.py --impl reference > $O/ref_n1.json 2> $O/ref_n1.err
echo done

#!/bin/bash
# round 2, one GPU: the faster GPU generator against the CPU one, the virtual-rank suite (C3 at W = 8 included),
# the graphed real producer (train c = 16 / c = 1), straggler calibration with graphed sub-batches.
set -x
O=gpurun_out/r2e
mkdir -p $O
python -m pytest tests/test_gpu_synth.py -q > $O/synth.log 2>&1
python -m pytest tests/test_gpu_virtual.py -q -s --durations=5 > $O/virtual.log 2>&1
python bench.py --mode train --steps 4 --warmup 2 > $O/train_n1_c16.json 2> $O/train_n1_c16.err
python bench.py --mode train --update-freq 1 --steps 20 --warmup 3 > $O/train_n1_c1.json 2> $O/train_n1_c1.err
python tools/straggler_calibrate.py --measure 240 --out $O/straggler_graphed.txt > $O/straggler.log 2>&1
echo done

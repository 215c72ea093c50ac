#!/bin/bash
set -x
O=gpurun_out/r2u
mkdir -p $O
timeout 300 python tools/repro_c1.py > $O/repro.log 2>&1
echo done

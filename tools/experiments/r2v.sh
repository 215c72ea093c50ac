#!/bin/bash
O=gpurun_out/r2v
mkdir -p $O
./tools/k1_stats_probe > $O/probe.log 2>&1
echo done

#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/red
B="python bench.py --steps 1 --warmup 3 --workload config3-default --angle-sets 1 --no-cpu-baseline --no-config5"
QTN_FUSE_MIN_POS=0 $B > gpurun_out/red/plain.log 2>&1; echo "plain rc=$?"
QTN_FUSE_MIN_POS=0 ncu --set full --clock-control none --import-source on -k regex:reduce_kernel -s 10 -c 1 -o gpurun_out/red/red $B > gpurun_out/red/ncu.log 2>&1; echo "ncu rc=$?"

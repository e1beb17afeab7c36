#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/c3d
B="python bench.py --steps 1 --warmup 3 --workload config3-default --angle-sets 1 --no-cpu-baseline --no-config5"
$B > gpurun_out/c3d/plain2.log 2>&1; echo "plain rc=$?"
ncu --set full --clock-control none --import-source on -k regex:stream_kernel -s ${SKIP:-20} -c 1 -o gpurun_out/c3d/big $B > gpurun_out/c3d/ncu2.log 2>&1; echo "ncu rc=$?"

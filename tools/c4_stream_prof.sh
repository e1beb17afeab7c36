#!/bin/bash
# ncu full capture of the first 24 stream_kernel launches of config 4 (pick the [2,16,26]->25 one by duration)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/c4
B="python bench.py --steps 1 --warmup 3 --workload config4 --angle-sets 1 --no-cpu-baseline --no-config5"
$B > gpurun_out/c4/plain.log 2>&1; echo "plain rc=$?"
ncu --set full --clock-control none -k regex:stream_kernel -s 10 -c 6 -o gpurun_out/c4/streams $B > gpurun_out/c4/ncu6.log 2>&1; echo "ncu6 rc=$?"

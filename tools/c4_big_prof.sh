#!/bin/bash
# ncu full captures of config 4's two largest launches: the [1,22,21]->26
# expanding bucket (expand_kernel, 8th launch) and the [2,16,26]->25 bucket
# (stream_kernel, 14th launch) of the first evaluation
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/c4
B="python bench.py --steps 1 --warmup 3 --workload config4 --angle-sets 1 --no-cpu-baseline --no-config5"
$B > gpurun_out/c4/plain.log 2>&1; echo "plain rc=$?"
ncu --set full --clock-control none --import-source on -k regex:expand_kernel -s 7 -c 1 -o gpurun_out/c4/big_expand $B > gpurun_out/c4/ncu3.log 2>&1; echo "ncu3 rc=$?"
[ -n "$STREAM" ] && ncu --set full --clock-control none --import-source on -k regex:stream_kernel -s 13 -c 1 -o gpurun_out/c4/big_stream $B > gpurun_out/c4/ncu4.log 2>&1; echo "ncu4 rc=$?"

#!/bin/bash
# full ncu capture of the config-4 expanding-bucket levels (15, 22, 26, 27)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/c4
B="python bench.py --steps 1 --warmup 3 --workload config4 --angle-sets 1 --no-cpu-baseline --no-config5"
$B > gpurun_out/c4/plain.log 2>&1; echo "plain rc=$?"
for s in ${C4_LEVELS:-26}; do
ncu --set full --clock-control none --import-source on -k regex:stream_kernel -s $s -c 1 -o gpurun_out/c4/lev$s $B > gpurun_out/c4/ncu$s.log 2>&1; echo "ncu $s rc=$?"
done

#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/c4
B="python bench.py --steps 1 --warmup 3 --workload config4 --angle-sets 1 --no-cpu-baseline --no-config5"
$B > gpurun_out/c4/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 80 --csv --log-file gpurun_out/c4/launches.csv $B > gpurun_out/c4/ncu.log 2>&1; echo "ncu rc=$?"
ncu --set full --clock-control none --import-source on -k regex:expand_kernel -c 12 -o gpurun_out/c4/prof_expand $B > gpurun_out/c4/ncu2.log 2>&1; echo "ncu2 rc=$?"

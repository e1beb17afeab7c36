#!/bin/bash
# config-3 default: per-level launch list (time, DRAM) of one evaluation
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/c3d
B="python bench.py --steps 1 --warmup 3 --workload config3-default --angle-sets 1 --no-cpu-baseline --no-config5"
$B > gpurun_out/c3d/plain.log 2>&1; echo "plain rc=$?"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size --clock-control none -c 320 --csv --log-file gpurun_out/c3d/launches.csv $B > gpurun_out/c3d/ncu.log 2>&1; echo "ncu rc=$?"

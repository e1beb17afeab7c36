#!/bin/bash
# Config 3 default: launch list with grid sizes, full capture of a long fused launch.
cd "$(dirname "$0")/.."
O=gpurun_out/${1:-c3d}; mkdir -p $O
B="python bench.py --steps 1 --warmup 3 --workload config3-default --angle-sets 1 --no-cpu-baseline --no-records"
$B > $O/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -c 200 --csv --log-file $O/launches.csv $B > $O/ncu_l.log 2>&1; echo "ncu launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:fused_kernel -s 27 -c 1 -o $O/prof_fused27 $B > $O/ncu_f.log 2>&1; echo "ncu fused rc=$?"

#!/bin/bash
# Set-major executor evidence: launch list (time + DRAM bytes) of the default
# config-2 bench step and a full capture of one evaluation's level launches.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/sm
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-config5"
$B > gpurun_out/sm/plain.log 2>&1; echo "plain rc=$?"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none -c 120 --csv --log-file gpurun_out/sm/launches_config2.csv $B > gpurun_out/sm/ncu1.log 2>&1; echo "ncu1 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:sm_ -c 24 -o gpurun_out/sm/prof_sm $B > gpurun_out/sm/ncu2.log 2>&1; echo "ncu2 rc=$?"

#!/bin/bash
# full ncu capture of the largest set-major level for two kernel variants
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/sm2
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-config5"
$B > gpurun_out/sm2/plain.log 2>&1; echo "plain rc=$?"
QTN_SM_BUCKET=1 ncu --set full --clock-control none --import-source on -k regex:sm_bucket -s 2 -c 1 -o gpurun_out/sm2/bucket $B > gpurun_out/sm2/ncu_b.log 2>&1; echo "ncu b rc=$?"
QTN_SM_BUCKET=0 ncu --set full --clock-control none --import-source on -k regex:sm_level -s 2 -c 1 -o gpurun_out/sm2/level $B > gpurun_out/sm2/ncu_l.log 2>&1; echo "ncu l rc=$?"

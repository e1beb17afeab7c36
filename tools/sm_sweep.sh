#!/bin/bash
# set-major executor over angle-set counts (config 2) and config 3; env variants
cd "$(dirname "$0")/.."
for v in ${SWEEP_VARS:-X=1}; do
echo "$v"
for A in 256 1024 2048; do
  env $v timeout 300 python bench.py --angle-sets $A --steps 10 --warmup 3 --no-cpu-baseline --no-config5 2>&1 | tail -1 | cut -c1-130
done
env $v timeout 300 python bench.py --workload config3 --angle-sets 1024 --steps 5 --warmup 3 --no-cpu-baseline --no-config5 2>&1 | tail -1 | cut -c1-130
env $v timeout 300 python bench.py --workload config3 --angle-sets 256 --steps 5 --warmup 3 --no-cpu-baseline --no-config5 2>&1 | tail -1 | cut -c1-130
done

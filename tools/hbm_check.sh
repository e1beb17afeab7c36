#!/bin/bash
# HBM-executor workloads: config 4, config 3 default, config 5 (w=30)
cd "$(dirname "$0")/.."
timeout 300 python bench.py --workload config4 --angle-sets 1 --steps 10 --warmup 3 --no-cpu-baseline --no-config5 2>&1 | tail -1 | cut -c1-140
timeout 300 python bench.py --workload config3-default --angle-sets 1 --steps 3 --warmup 3 --no-cpu-baseline --no-config5 2>&1 | tail -1 | cut -c1-140
timeout 300 python bench.py --workload config5 --steps 5 --c5-ws 26,30 --c5-ms 4,16 2>&1 | cut -c1-100

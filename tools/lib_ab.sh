#!/bin/bash
# A/B of an alternative build (QTN_LIB) on the HBM workloads and config 5
cd "$(dirname "$0")/.."
for lib in "" "$ALT_LIB"; do
  echo "lib=$lib"
  QTN_LIB=$lib timeout 300 python bench.py --workload config4 --angle-sets 1 --steps 10 --warmup 3 --no-cpu-baseline --no-config5 2>&1 | tail -1 | cut -c1-100
  QTN_LIB=$lib timeout 300 python bench.py --workload config3-default --angle-sets 1 --steps 3 --warmup 3 --no-cpu-baseline --no-config5 2>&1 | tail -1 | cut -c1-100
  QTN_LIB=$lib timeout 300 python bench.py --workload config5 --steps 5 --c5-ws 26,30 --c5-ms 4,16 2>&1 | cut -c1-90
done

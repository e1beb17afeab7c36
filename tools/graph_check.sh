#!/bin/bash
cd "$(dirname "$0")/.."
for g in 1 0; do
  echo "QTN_GRAPHS=$g"
  for A in 1 128 1024; do QTN_GRAPHS=$g timeout 300 python bench.py --angle-sets $A --steps 10 --warmup 3 --no-cpu-baseline --no-config5 2>&1 | tail -1 | cut -c1-100; done
  QTN_GRAPHS=$g timeout 300 python bench.py --workload config4 --angle-sets 1 --steps 10 --warmup 3 --no-cpu-baseline --no-config5 2>&1 | tail -1 | cut -c1-100
  QTN_GRAPHS=$g timeout 300 python bench.py --workload config3-default --angle-sets 1 --steps 3 --warmup 3 --no-cpu-baseline --no-config5 2>&1 | tail -1 | cut -c1-100
done

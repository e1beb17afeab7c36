#!/bin/bash
# One GPU session: GPU tests, smoke, the default bench line and the reference arm.
cd "$(dirname "$0")/.."
O=gpurun_out/${1:-chk}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
timeout 1200 python -m pytest tests -q -m gpu -rA > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 python __graft_entry__.py > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err; echo "ref rc=$?"

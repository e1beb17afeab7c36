set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
for e in 64 1000000000; do
QTN_SETMAJOR_MIN_SETS=$e timeout 300 python bench.py --steps 10 --warmup 3 2>&1 | tail -1
QTN_SETMAJOR_MIN_SETS=$e timeout 300 python bench.py --workload config3 --angle-sets 256 --steps 5 --warmup 3 2>&1 | tail -1
done

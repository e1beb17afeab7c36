mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -4 gpurun_out/pytest_gpu.log
for S in 1 2 4 8; do QTN_SETS_PER_WARP=$S timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-config5 > gpurun_out/b_S$S.json 2>&1; echo S=$S rc=$?; done
for S in 1 2 4; do QTN_SETS_PER_WARP=$S timeout 300 python bench.py --workload config3 --angle-sets 256 --steps 5 --warmup 3 --no-cpu-baseline --no-config5 > gpurun_out/b_c3_S$S.json 2>&1; echo c3 rc=$?; done

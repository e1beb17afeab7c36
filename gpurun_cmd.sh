mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_gpu.log
for Lv in 0 8 32; do QTN_LANES_PER_SET=$Lv timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-config5 > gpurun_out/b_L$Lv.json 2>&1; done
for Lv in 0 16; do QTN_LANES_PER_SET=$Lv timeout 300 python bench.py --workload config3 --angle-sets 256 --steps 5 --warmup 3 --no-cpu-baseline --no-config5 > gpurun_out/b_c3_L$Lv.json 2>&1; done

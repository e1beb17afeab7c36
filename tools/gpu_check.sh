mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -4 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --workload config5 --steps 5 --c5-ws 28,30 --c5-ms 4,16 > gpurun_out/c5_sweep.json 2>&1; echo c5 rc=$?
timeout 300 python bench.py --steps 5 --warmup 3 --workload config4 --angle-sets 1 --no-config5 --no-cpu-baseline > gpurun_out/b_c4.json 2>&1; echo c4 rc=$?
timeout 300 python bench.py --steps 3 --warmup 3 --workload config3-default --angle-sets 1 --no-config5 --no-cpu-baseline > gpurun_out/b_c3d.json 2>&1; echo c3d rc=$?

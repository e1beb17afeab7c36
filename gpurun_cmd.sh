mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -4 gpurun_out/pytest_gpu.log
for k in 0 3 6; do timeout 300 python bench.py --steps 5 --warmup 3 --workload config4 --angle-sets 1 --slices $k --no-config5 --no-cpu-baseline > gpurun_out/b_c4_k$k.json 2>&1; echo c4 k=$k rc=$?; done
timeout 300 python bench.py --steps 5 --warmup 3 --workload config4 --angle-sets 8 --slices 3 --no-config5 --no-cpu-baseline > gpurun_out/b_c4_k3_A8.json 2>&1; echo c4 A8 rc=$?
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/b_default.json 2>&1; echo default rc=$?

mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -x -k "expand or config4" > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --workload config4 --angle-sets 1 --steps 10 --warmup 3 --no-config5 --no-cpu-baseline > gpurun_out/b_c4.json 2>&1; echo c4 rc=$?
python -c "import json; d=json.loads(open('gpurun_out/b_c4.json').read().strip().splitlines()[-1]); print('c4', d['value'], d['ms_per_step'], d['config']['energy_set0'])"
timeout 300 python bench.py --workload config3-default --angle-sets 1 --steps 5 --warmup 3 --no-config5 --no-cpu-baseline > gpurun_out/b_c3d.json 2>&1; echo c3d rc=$?
python -c "import json; d=json.loads(open('gpurun_out/b_c3d.json').read().strip().splitlines()[-1]); print('c3d', d['value'], d['ms_per_step'], d['config']['energy_set0'])"
B="python bench.py --steps 1 --warmup 3 --workload config4 --angle-sets 1 --no-cpu-baseline --no-config5"
mkdir -p gpurun_out/c4; [ -n "$PROF" ] && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 80 --csv --log-file gpurun_out/c4/launches.csv $B > gpurun_out/c4/ncu.log 2>&1; echo "ncu rc=$?"

mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -x -k "setmajor or config2" > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
for x in 0 1; do
QTN_SM_PAIR=$x timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-config5 > gpurun_out/b_c2_$x.json 2>&1; echo rc=$?
python -c "import json; d=json.loads(open('gpurun_out/b_c2_$x.json').read().strip().splitlines()[-1]); print('c2 pair=$x', d['value'], d['roofline']['avg_launch_s'], d['e2e']['value'], d['config']['energy_set0'])"
QTN_SM_PAIR=$x timeout 300 python bench.py --workload config3 --angle-sets 256 --steps 10 --warmup 3 --no-cpu-baseline --no-config5 > gpurun_out/b_c3_$x.json 2>&1; echo rc=$?
python -c "import json; d=json.loads(open('gpurun_out/b_c3_$x.json').read().strip().splitlines()[-1]); print('c3 pair=$x', d['value'], d['roofline']['avg_launch_s'], d['config']['energy_set0'])"
done

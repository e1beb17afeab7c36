mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -x -k "setmajor" > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_gpu.log
for x in 0 1; do
QTN_SM_BULK=$x timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-config5 > gpurun_out/b_c2_$x.json 2>&1; echo rc=$?
python -c "import json; d=json.loads(open('gpurun_out/b_c2_$x.json').read().strip().splitlines()[-1]); print('c2 bulk=$x', d['value'], d['roofline']['avg_launch_s'], d['config']['energy_set0'])"
QTN_SM_BULK=$x timeout 300 python bench.py --workload config3 --angle-sets 256 --steps 10 --warmup 3 --no-cpu-baseline --no-config5 > gpurun_out/b_c3_$x.json 2>&1; echo rc=$?
python -c "import json; d=json.loads(open('gpurun_out/b_c3_$x.json').read().strip().splitlines()[-1]); print('c3 bulk=$x', d['value'], d['roofline']['avg_launch_s'], d['config']['energy_set0'])"
done
for m in 60000 150000; do for c in 148 296 444; do
QTN_SM_BULK_SMEM=$m QTN_SM_BULK_CTAS=$c timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-config5 > gpurun_out/b_c2_t.json 2>&1
python -c "import json; d=json.loads(open('gpurun_out/b_c2_t.json').read().strip().splitlines()[-1]); print('c2 smem=$m ctas=$c', d['value'], d['roofline']['avg_launch_s'])"
done; done

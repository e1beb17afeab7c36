mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -x -k "expand or config4 or config3_default" > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/pytest_gpu.log
for x in 0 1; do
QTN_EXPAND=$x timeout 300 python bench.py --workload config4 --angle-sets 1 --steps 10 --warmup 3 --no-config5 --no-cpu-baseline > gpurun_out/b_c4_$x.json 2>&1; echo c4 rc=$?
python -c "import json; d=json.loads(open('gpurun_out/b_c4_$x.json').read().strip().splitlines()[-1]); print('c4 x=$x', d['value'], d['ms_per_step'], d['config']['energy_set0'])"
QTN_EXPAND=$x timeout 300 python bench.py --workload config3-default --angle-sets 1 --steps 5 --warmup 3 --no-config5 --no-cpu-baseline > gpurun_out/b_c3d_$x.json 2>&1; echo c3d rc=$?
python -c "import json; d=json.loads(open('gpurun_out/b_c3d_$x.json').read().strip().splitlines()[-1]); print('c3d x=$x', d['value'], d['ms_per_step'], d['config']['energy_set0'])"
done

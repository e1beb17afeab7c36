mkdir -p gpurun_out
[ -z "$NOTEST" ] && timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
for x in 0 1; do
QTN_FUSE_REDUCE=$x timeout 300 python bench.py --workload config4 --angle-sets 1 --steps 10 --warmup 3 --no-config5 --no-cpu-baseline > gpurun_out/b_c4_$x.json 2>&1; echo c4 rc=$?
python -c "import json; d=json.loads(open('gpurun_out/b_c4_$x.json').read().strip().splitlines()[-1]); print('c4 fuse=$x', d['value'], d['ms_per_step'], d['gpu_launches'], d['config']['energy_set0'])"
QTN_FUSE_REDUCE=$x timeout 300 python bench.py --workload config3-default --angle-sets 1 --steps 5 --warmup 3 --no-config5 --no-cpu-baseline > gpurun_out/b_c3d_$x.json 2>&1; echo c3d rc=$?
python -c "import json; d=json.loads(open('gpurun_out/b_c3d_$x.json').read().strip().splitlines()[-1]); print('c3d fuse=$x', d['value'], d['ms_per_step'], d['gpu_launches'], d['config']['energy_set0'])"
done

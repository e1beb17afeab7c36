mkdir -p gpurun_out
for tb in 9 6 3; do
QTN_XMIN_TILE_BITS=$tb timeout 300 python bench.py --workload config4 --angle-sets 1 --steps 10 --warmup 3 --no-config5 --no-cpu-baseline > gpurun_out/b_c4.json 2>&1
python -c "import json; d=json.loads(open('gpurun_out/b_c4.json').read().strip().splitlines()[-1]); print('c4 tb=$tb', d['value'], d['ms_per_step'], d['config']['energy_set0'])"
QTN_XMIN_TILE_BITS=$tb timeout 300 python bench.py --workload config3-default --angle-sets 1 --steps 5 --warmup 3 --no-config5 --no-cpu-baseline > gpurun_out/b_c3d.json 2>&1
python -c "import json; d=json.loads(open('gpurun_out/b_c3d.json').read().strip().splitlines()[-1]); print('c3d tb=$tb', d['value'], d['ms_per_step'], d['config']['energy_set0'])"
done

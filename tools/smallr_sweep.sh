for r in 9 10 11 12 13; do
QTN_SMALL_R=$r timeout 300 python bench.py --workload config3-default --angle-sets 1 --steps 5 --warmup 3 --no-config5 --no-cpu-baseline > /tmp/b.json 2>&1
python -c "import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print('c3d small_r=$r', d['value'], d['ms_per_step'], d['gpu_launches'], d['config']['energy_set0'])"
QTN_SMALL_R=$r timeout 300 python bench.py --workload config4 --angle-sets 1 --steps 10 --warmup 3 --no-config5 --no-cpu-baseline > /tmp/b.json 2>&1
python -c "import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print('c4 small_r=$r', d['value'], d['ms_per_step'], d['gpu_launches'], d['config']['energy_set0'])"
done

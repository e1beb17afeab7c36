timeout 600 python -m pytest tests -q -m gpu -x -k "setmajor" 2>&1 | tail -1
for al in 2 3; do
QTN_SM_ALIGN=$al timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-config5 > /tmp/b.json 2>&1
python -c "import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print('align=$al c2', d['value'], d['roofline']['avg_launch_s'])"
QTN_SM_ALIGN=$al timeout 300 python bench.py --workload config3 --angle-sets 256 --steps 20 --warmup 5 --no-cpu-baseline --no-config5 > /tmp/b.json 2>&1
python -c "import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print('align=$al c3', d['value'], d['roofline']['avg_launch_s'])"
done

timeout 600 python -m pytest tests -q -m gpu -x -k "setmajor" 2>&1 | tail -1
for A in 128 256 512 1024; do
timeout 300 python bench.py --workload config3 --angle-sets $A --steps 10 --warmup 3 --no-cpu-baseline --no-config5 > /tmp/b.json 2>&1
python -c "import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print('c3 A=$A', d['value'], d['roofline']['frac'])"
timeout 300 python bench.py --angle-sets $A --steps 10 --warmup 3 --no-cpu-baseline --no-config5 > /tmp/b.json 2>&1
python -c "import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print('c2 A=$A', d['value'], d['roofline']['frac'])"
done

# A/B of the in-tree build against build_alt/libqtn_base.so on config 1 (complex128, 1024 angle sets), 3 rounds
cd "$(dirname "$0")/.."
for rep in 1 2 3; do
for lib in "" "$PWD/build_alt/libqtn_base.so"; do
  QTN_LIB=$lib timeout 300 python bench.py --workload config1 --angle-sets 1024 --steps 20 --warmup 5 --no-config5 --no-cpu-baseline > /tmp/b.json 2>&1
  python -c "import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print('config1 ${lib:-intree}', round(d['value']/1e6,2), round(d['ms_per_step'],4))"
done; done

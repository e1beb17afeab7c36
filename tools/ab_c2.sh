# A/B of alternative builds (ALT_LIBS = file names under build_alt/) on config 2 (default bench), 3 rounds
cd "$(dirname "$0")/.."
for rep in 1 2 3; do
for lib in "" $(for a in $ALT_LIBS; do echo "$PWD/build_alt/$a"; done); do
  QTN_LIB=$lib timeout 300 python bench.py --steps 20 --warmup 5 --no-config5 --no-cpu-baseline > /tmp/b.json 2>&1
  python -c "import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print('config2 ${lib:-intree}', round(d['value']/1e6,2), round(d['ms_per_step'],4), d['config']['energy_set0'])"
done; done

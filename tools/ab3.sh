# A/B of alternative builds (ALT_LIBS = file names under build_alt/) on config 4 and config 3 default, 2 rounds
cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests -q -m gpu -x -k "trace or config4 or staged" 2>&1 | tail -1
run() {
  QTN_LIB=$1 timeout 300 python bench.py --workload $2 --angle-sets 1 --steps $3 --warmup 3 --no-config5 --no-cpu-baseline > /tmp/b.json 2>&1
  python -c "import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print('$2 ${1:-intree}', round(d['value'],1), round(d['ms_per_step'],4), d['config']['energy_set0'])"
}
for rep in 1 2; do
for lib in "$PWD/build_alt/libqtn_base.so" "" $(for a in $ALT_LIBS; do echo "$PWD/build_alt/$a"; done); do
  run "$lib" config4 20
  run "$lib" config3-default 5
done; done

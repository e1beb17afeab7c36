# A/B of environment settings on config 4 and config 3 default (interleaved, 2 rounds); ENVS="A=1 B=2 ..."
cd "$(dirname "$0")/.."
[ -n "$TESTS" ] && timeout 600 python -m pytest tests -q -m gpu -x $TESTS 2>&1 | tail -1
run() {
  env $1 timeout 300 python bench.py --workload $2 --angle-sets 1 --steps $3 --warmup 3 --no-config5 --no-cpu-baseline > /tmp/b.json 2>&1
  python -c "import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print('$2 $1', round(d['value'],1), round(d['ms_per_step'],4), d['gpu_launches'], d['config']['energy_set0'])"
}
for rep in 1 2; do
for e in $ENVS; do
  run "$e" config4 20
  run "$e" config3-default 5
done; done

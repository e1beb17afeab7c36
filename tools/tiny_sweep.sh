# HBM-executor routing sweep: QTN_TINY_LEVEL / QTN_SMALL_R on config 4 and config 3 default
mkdir -p gpurun_out
QTN_DEBUG_ROUTE=1 timeout 300 python bench.py --workload config4 --angle-sets 1 --steps 2 --warmup 3 --no-config5 --no-cpu-baseline 2>&1 | grep stream-item | sort | uniq -c
run() {  # env workload steps
  env $1 timeout 300 python bench.py --workload $2 --angle-sets 1 --steps $3 --warmup 3 --no-config5 --no-cpu-baseline > /tmp/b.json 2>&1
  python -c "import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print('$2 $1', round(d['value'],1), round(d['ms_per_step'],4), d['gpu_launches'], d['config']['energy_set0'])"
}
for e in QTN_X=0 QTN_TINY_LEVEL=524288 QTN_TINY_LEVEL=2097152 QTN_TINY_LEVEL=8388608 QTN_SMALL_R=14 QTN_SMALL_R=18 QTN_SMALL_R=20; do
  run $e config4 10
  run $e config3-default 5
done

# quick GPU iteration: selected tests (-k "$1"), the default bench line, extra bench args in $2
mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -x ${1:+-k "$1"} > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-config5 $2 > gpurun_out/bench_iter.json 2> gpurun_out/bench_iter.err; echo bench rc=$?
cat gpurun_out/bench_iter.json; tail -3 gpurun_out/bench_iter.err

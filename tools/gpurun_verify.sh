set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/v_pytest_gpu.log 2>&1; echo pytest rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v_smoke.log 2>&1; echo smoke rc=$?
timeout 400 python bench.py > gpurun_out/v_bench_default.json 2>gpurun_out/v_bench_default.err; echo bench rc=$?
timeout 400 python bench.py --impl reference > gpurun_out/v_bench_ref.json 2>gpurun_out/v_bench_ref.err; echo ref rc=$?
tail -3 gpurun_out/v_pytest_gpu.log; tail -2 gpurun_out/v_smoke.log; cat gpurun_out/v_bench_default.json gpurun_out/v_bench_ref.json

timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/b_default.json 2>&1; echo default rc=$?

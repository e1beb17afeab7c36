mkdir -p gpurun_out
python bench.py --workload config5 --steps 5 --c5-ws 26,28,30,32 --c5-ms 4,16 > gpurun_out/c5_sweep.json 2>&1; echo c5 rc=$?
python bench.py --steps 10 --warmup 3 > gpurun_out/b_default.json 2> gpurun_out/b_default.err; echo default rc=$?
python bench.py --workload config5 --steps 2 --c5-ws 28 --c5-ms 16 > gpurun_out/plain_c5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:bucket_kernel -s 2 -c 1 -o gpurun_out/prof_c5_w28 python bench.py --workload config5 --steps 2 --c5-ws 28 --c5-ms 16 > gpurun_out/ncu_c5.log 2>&1; echo ncu1 rc=$?
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-config5 > gpurun_out/plain_c2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:smem_net -s 3 -c 1 -o gpurun_out/prof_smem python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-config5 > gpurun_out/ncu_smem.log 2>&1; echo ncu2 rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-config5 > gpurun_out/ncu_launch.log 2>&1; echo ncu3 rc=$?

#!/bin/bash
# One GPU session: tests, smoke, the default bench line, the reference arm,
# the other workloads, the config-5 roofline sweep and the ncu evidence.
mkdir -p gpurun_out/r
cd "$(dirname "$0")/.."
timeout 1200 python -m pytest tests -q -m gpu -rA > gpurun_out/r/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 python __graft_entry__.py > gpurun_out/r/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/r/bench_default.json 2> gpurun_out/r/bench_default.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r/bench_reference.json 2>&1; echo "ref rc=$?"
timeout 300 python bench.py --workload config1 --angle-sets 1024 --steps 50 --warmup 10 --no-records --cpu-seconds 5 > gpurun_out/r/bench_config1.json 2>&1; echo "c1 rc=$?"
timeout 300 python bench.py --workload config3 --angle-sets 256 --steps 5 --warmup 3 --no-records --cpu-seconds 5 > gpurun_out/r/bench_config3.json 2>&1; echo "c3 rc=$?"
timeout 300 python bench.py --workload config3-default --angle-sets 1 --steps 20 --warmup 5 --no-records --cpu-seconds 10 > gpurun_out/r/bench_config3d.json 2>&1; echo "c3d rc=$?"
timeout 300 python bench.py --workload config4 --angle-sets 1 --steps 10 --warmup 3 --no-records --cpu-seconds 20 > gpurun_out/r/bench_config4.json 2>&1; echo "c4 rc=$?"
timeout 300 python bench.py --workload config4 --angle-sets 1 --slices 3 --steps 10 --warmup 3 --no-records --no-cpu-baseline > gpurun_out/r/bench_config4_k3.json 2>&1; echo "c4k3 rc=$?"
timeout 600 python bench.py --workload config5 --steps 5 > gpurun_out/r/config5_sweep.json 2>&1; echo "c5 rc=$?"
# ncu: launch list of the default bench step, then full captures of the two hot kernels
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-records > gpurun_out/r/plain_c2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/r/launches_config2.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-records > gpurun_out/r/ncu1.log 2>&1; echo "ncu1 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:sm_level_kernel -c 15 -o gpurun_out/r/prof_setmajor python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-records > gpurun_out/r/ncu2.log 2>&1; echo "ncu2 rc=$?"
python bench.py --steps 3 --warmup 3 --angle-sets 16 --no-cpu-baseline --no-records > gpurun_out/r/plain_c2_16.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:smem_net -s 3 -c 1 -o gpurun_out/r/prof_smem python bench.py --steps 3 --warmup 3 --angle-sets 16 --no-cpu-baseline --no-records > gpurun_out/r/ncu2b.log 2>&1; echo "ncu2b rc=$?"
python bench.py --workload config5 --steps 2 --c5-ws 30 --c5-ms 16 > gpurun_out/r/plain_c5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:stream_kernel -s 2 -c 1 -o gpurun_out/r/prof_stream_c5 python bench.py --workload config5 --steps 2 --c5-ws 30 --c5-ms 16 > gpurun_out/r/ncu3.log 2>&1; echo "ncu3 rc=$?"
python bench.py --steps 2 --warmup 3 --workload config4 --angle-sets 1 --no-cpu-baseline --no-records > gpurun_out/r/plain_c4.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 80 --csv --log-file gpurun_out/r/launches_config4.csv python bench.py --steps 2 --warmup 3 --workload config4 --angle-sets 1 --no-cpu-baseline --no-records > gpurun_out/r/ncu4.log 2>&1; echo "ncu4 rc=$?"
# the largest chain of config 4 ([1,22,21] -> 26, its consumer [2,16,26] -> 25 and three traces -> 22: the 6th xt launch)
ncu --set full --clock-control none --import-source on -k regex:xt_kernel -s 5 -c 1 -o gpurun_out/r/prof_xt_c4 python bench.py --steps 2 --warmup 3 --workload config4 --angle-sets 1 --no-cpu-baseline --no-records > gpurun_out/r/ncu5.log 2>&1; echo "ncu5 rc=$?"
# the tail chain of config 4 (rank-22 intermediate -> scalar as one weighted sum)
ncu --set full --clock-control none --import-source on -k regex:wsum_kernel -s 3 -c 1 -f -o gpurun_out/r/prof_wsum_c4 python bench.py --steps 2 --warmup 3 --workload config4 --angle-sets 1 --no-cpu-baseline --no-records > gpurun_out/r/ncu5b.log 2>&1; echo "ncu5b rc=$?"
python tools/micro/write_bw.py > gpurun_out/r/write_bw.txt 2>&1; echo "wbw rc=$?"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 320 --csv --log-file gpurun_out/r/launches_config3d.csv python bench.py --steps 1 --warmup 3 --workload config3-default --angle-sets 1 --no-cpu-baseline --no-records > gpurun_out/r/ncu6.log 2>&1; echo "ncu6 rc=$?"
for w in config4 config3-default; do timeout 300 python tools/timeline.py $w --out gpurun_out/r/timeline_$w.json > gpurun_out/r/timeline_$w.txt 2>&1; done
QTN_XT=0 timeout 300 python bench.py --workload config3-default --angle-sets 1 --steps 10 --warmup 3 --no-records --no-cpu-baseline > gpurun_out/r/bench_config3d_noxt.json 2>&1; echo "c3d noxt rc=$?"
QTN_XT=0 timeout 300 python bench.py --workload config4 --angle-sets 1 --steps 10 --warmup 3 --no-records --no-cpu-baseline > gpurun_out/r/bench_config4_noxt.json 2>&1; echo "c4 noxt rc=$?"
QTN_WSUM=0 timeout 300 python bench.py --workload config4 --angle-sets 1 --steps 10 --warmup 3 --no-records --no-cpu-baseline > gpurun_out/r/bench_config4_nowsum.json 2>&1; echo "c4 nowsum rc=$?"
QTN_WSUM=0 timeout 300 python bench.py --workload config3-default --angle-sets 1 --steps 10 --warmup 3 --no-records --no-cpu-baseline > gpurun_out/r/bench_config3d_nowsum.json 2>&1; echo "c3d nowsum rc=$?"
python bench.py --steps 1 --warmup 3 --workload config3-default --angle-sets 1 --no-cpu-baseline --no-records > gpurun_out/r/plain_c3d_f.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fused_kernel -s 20 -c 1 -o gpurun_out/r/prof_fused_c3d python bench.py --steps 1 --warmup 3 --workload config3-default --angle-sets 1 --no-cpu-baseline --no-records > gpurun_out/r/ncu7.log 2>&1; echo "ncu7 rc=$?"

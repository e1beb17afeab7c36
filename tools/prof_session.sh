#!/bin/bash
# Profiling session: in-graph timelines of config 4 / config 3 default and
# ncu --set full captures of the config-4 expanding bucket and a head small level.
cd "$(dirname "$0")/.."
O=gpurun_out/${1:-prof}; mkdir -p $O
for w in config4 config3-default; do timeout 300 python tools/timeline.py $w --out $O/timeline_$w.json > $O/timeline_$w.txt 2>&1; done
B="python bench.py --steps 1 --warmup 3 --workload config4 --angle-sets 1 --no-cpu-baseline --no-records"
$B > $O/plain_c4.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file $O/launches_config4.csv $B > $O/ncu_l4.log 2>&1; echo "ncu launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:expand_kernel -s 6 -c 1 -o $O/prof_expand_c4 $B > $O/ncu_x.log 2>&1; echo "ncu expand rc=$?"
ncu --set full --clock-control none --import-source on -k regex:small_kernel -s 4 -c 1 -o $O/prof_small_c4 $B > $O/ncu_s.log 2>&1; echo "ncu small rc=$?"
ncu --set full --clock-control none --import-source on -k regex:trace_kernel -s 4 -c 1 -o $O/prof_trace_c4 $B > $O/ncu_t.log 2>&1; echo "ncu trace rc=$?"

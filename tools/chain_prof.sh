mkdir -p gpurun_out/c4
B="python bench.py --steps 1 --warmup 3 --workload config4 --angle-sets 1 --no-cpu-baseline --no-config5"
QTN_CHAIN_ELEMS=4096 $B > /dev/null 2>&1
QTN_CHAIN_ELEMS=4096 ncu --set full --clock-control none -k regex:chain_kernel -c 2 -o gpurun_out/c4/chain $B > gpurun_out/c4/ncu_chain.log 2>&1; echo rc=$?
QTN_CHAIN_ELEMS=4096 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/c4/launches_chain.csv $B > /dev/null 2>&1; echo rc=$?

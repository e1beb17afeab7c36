mkdir -p gpurun_out
for LZ in 1 0; do for Lv in 4 8 16 32; do QTN_SMEM_LAZY=$LZ QTN_LANES_PER_SET=$Lv timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-config5 > gpurun_out/b_z${LZ}_L$Lv.json 2>&1; done; done
for LZ in 1 0; do for Lv in 16 32; do QTN_SMEM_LAZY=$LZ QTN_LANES_PER_SET=$Lv timeout 300 python bench.py --workload config3 --angle-sets 256 --steps 5 --warmup 3 --no-cpu-baseline --no-config5 > gpurun_out/b_c3_z${LZ}_L$Lv.json 2>&1; done; done

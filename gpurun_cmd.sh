mkdir -p gpurun_out
for V in default s8_t10 s6_t10 s3_t11; do
  if [ $V != default ]; then export QTN_LIB=$PWD/build_alt/lib_$V.so; fi
  echo "== $V" >> gpurun_out/ab.txt
  python tools/bucket_bench.py "P=27;G=0:0:0;T=1" "P=22;G=21:5:6;T=1" "P=22;G=12:5:2;T=1" >> gpurun_out/ab.txt 2>&1
  timeout 300 python bench.py --workload config5 --steps 5 --c5-ws 30 --c5-ms 4,16 >> gpurun_out/ab.txt 2>&1
  timeout 300 python bench.py --steps 5 --warmup 3 --workload config4 --angle-sets 1 --no-config5 --no-cpu-baseline > gpurun_out/b_c4_$V.json 2>&1
  python -c "import json; d=json.load(open('gpurun_out/b_c4_$V.json')); print('c4', d['ms_per_step'], d['config']['energy_set0'])" >> gpurun_out/ab.txt 2>&1
done

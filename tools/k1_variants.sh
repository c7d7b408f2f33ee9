# K1 throughput per instruction-mix variant (small config-5 slice), then ncu of variant 4.
SMALL="python bench.py --instances 296 --sweeps-per-step 100 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
for v in 0 2 4 6; do
  if [ $v = 0 ]; then LP=""; else LP="paper_2509_23043_b200/lib/variants/libtapt_v$v.so"; fi
  TAPT_LIB_PATH=$LP $SMALL > gpurun_out/smallv$v.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/smallv$v.json'));print('variant $v', d['value']/1e9, d['roofline']['kernel_ms_per_launch'])"
done
export TAPT_LIB_PATH=paper_2509_23043_b200/lib/variants/libtapt_v4.so
$SMALL > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k1_lattice -s 3 -c 1 -o gpurun_out/prof_k1_v4 -f $SMALL > gpurun_out/ncu_k1.log 2>&1; tail -1 gpurun_out/ncu_k1.log

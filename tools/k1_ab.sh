# A/B of library builds on the config-5 slice: bash tools/k1_ab.sh "12 100"
SMALL="python bench.py --instances 296 --sweeps-per-step 100 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
for v in $1; do
  for rep in 1 2; do
    TAPT_LIB_PATH=paper_2509_23043_b200/lib/variants/libtapt_v$v.so $SMALL > gpurun_out/ab_v$v.json 2>&1
    python -c "import json;d=json.load(open('gpurun_out/ab_v$v.json'));print('build $v', round(d['value']/1e9,1), round(d['roofline']['kernel_ms_per_launch'],2), round(d['roofline']['probe_ceiling']['value'],1))" || tail -3 gpurun_out/ab_v$v.json
  done
done

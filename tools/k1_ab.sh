# A/B of library builds on the config-5 slice: bash tools/k1_ab.sh "base um0"
# (base = lib/libtapt_b200.so, NAME = lib/variants/libtapt_NAME.so from tools/build_variant.sh)
SMALL="python bench.py --instances 296 --sweeps-per-step 100 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
for v in $1; do
  LP=paper_2509_23043_b200/lib/variants/libtapt_$v.so; [ "$v" = base ] && LP=paper_2509_23043_b200/lib/libtapt_b200.so
  for rep in 1 2; do
    TAPT_LIB_PATH=$LP $SMALL > gpurun_out/ab_$v.json 2>&1
    python -c "import json;d=json.load(open('gpurun_out/ab_$v.json'));print('build $v', round(d['value']/1e9,1), round(d['roofline']['kernel_ms_per_launch'],2), round(d['roofline']['probe_ceiling']['value'],1))" || tail -3 gpurun_out/ab_$v.json
  done
done

# K1 throughput per (instruction-mix variant, launch shape) on a small config-5 slice.
# usage: bash tools/k1_variants.sh "4 12" "512 256"
VARIANTS=${1:-"4"}
THREADS=${2:-"512"}
SMALL="python bench.py --instances 296 --sweeps-per-step 100 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
for v in $VARIANTS; do
  for nt in $THREADS; do
    LP="paper_2509_23043_b200/lib/variants/libtapt_v$v.so"
    TAPT_K1_THREADS=$nt TAPT_LIB_PATH=$LP $SMALL > gpurun_out/small_v${v}_t$nt.json 2>&1
    python -c "import json;d=json.load(open('gpurun_out/small_v${v}_t$nt.json'));print('variant $v threads $nt', round(d['value']/1e9,1), round(d['roofline']['kernel_ms_per_launch'],2))" || tail -3 gpurun_out/small_v${v}_t$nt.json
  done
done

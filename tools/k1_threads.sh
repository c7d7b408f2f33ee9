# K1 launch shapes on the config-5 slice
SMALL="python bench.py --instances 296 --sweeps-per-step 100 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
for nt in $1; do
  TAPT_K1_THREADS=$nt $SMALL > gpurun_out/small_t$nt.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/small_t$nt.json'));print('threads $nt', round(d['value']/1e9,1), round(d['roofline']['kernel_ms_per_launch'],2))" || tail -3 gpurun_out/small_t$nt.json
done

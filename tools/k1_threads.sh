# K1 launch-shape comparison on the small config-5 slice + GPU parity suite.
python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
SMALL="python bench.py --instances 296 --sweeps-per-step 100 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
for nt in 512 1024 768; do
  TAPT_K1_THREADS=$nt $SMALL > gpurun_out/small_t$nt.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/small_t$nt.json'));print('threads $nt', d['value']/1e9, d['roofline']['kernel_ms_per_launch'], d['roofline']['probe_ceiling']['value'])"
done

# Per-GPU throughput at the shard sizes of N = 8/4/2/1 (4096 instances strong-scaled), one GPU.
for I in 512 1024 2048 4096; do
  python bench.py --instances $I --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/shard_$I.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/shard_$I.json'));print('instances $I', round(d['value']/1e9,1), 'G/s, kernel', round(d['roofline']['achieved'],1))" || tail -3 gpurun_out/shard_$I.json
done

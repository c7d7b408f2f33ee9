# K2 launch-shape sweep on config 4 (threads x instances per CTA): bash tools/k2_shapes.sh "128 256 512" "1 2"
for nt in ${1:-256 512 1024}; do for ipb in ${2:-1 2 4}; do
  r=$(TAPT_K2_THREADS=$nt TAPT_K2_IPB=$ipb python tools/bench_configs.py --configs 4 2>/dev/null | python -c "import json,sys; print(round(json.loads(sys.stdin.read())['updates_per_s']/1e9,1))")
  echo "threads $nt ipb $ipb -> $r G/s"
done; done

# K3 instance teams per CTA on config 4 (ipb = 3 gives 444 co-resident teams < 512 instances: balanced schedule)
for ipb in 4 3 2 1; do
  echo "TAPT_K3_IPB=$ipb $(TAPT_K3_IPB=$ipb python tools/bench_configs.py --configs 4 --steps 2 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["kernel"], round(d["updates_per_s"]/1e9,1), "G/s", "success", d.get("coldest_slot_success"))')"
done

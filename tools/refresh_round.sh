# Round evidence in one call: tools/profile_round.sh (bench, launch list, K1 ncu), bench.py --workload cfg1..4,
# tools/bench_configs.py; then python tools/update_profiles.py copies the results into profiles/.
bash tools/profile_round.sh > gpurun_out/profile_round.log 2>&1
for k in 1 2 3 4; do python bench.py --workload cfg$k 2>/dev/null | tail -1; done > gpurun_out/workloads.jsonl
python tools/bench_configs.py --configs 1,2,3,4 --steps 2 > gpurun_out/configs.jsonl 2>&1
python tools/ncu_summary.py gpurun_out/prof_k1.ncu-rep k1_lattice > gpurun_out/k1_summary.txt 2>&1
tail -c 400 gpurun_out/bench_default.json; wc -l gpurun_out/workloads.jsonl gpurun_out/launches.csv

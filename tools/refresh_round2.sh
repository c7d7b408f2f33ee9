# Round-2 evidence in one GPU call: headline bench + launch list + K1 ncu (tools/profile_round.sh),
# the per-config lines (bench.py --workload cfg1..4), K3 ncu (tools/profile_k3.sh), the IsingFormer
# engines (tools/bench_former.py, tools/profile_former_tc.sh) and the full-length runs of the five
# configs (tools/run_configs.py).  Then: python tools/update_profiles.py --round 02
bash tools/refresh_round.sh > gpurun_out/refresh.log 2>&1
bash tools/profile_k3.sh > gpurun_out/profile_k3.log 2>&1
python tools/bench_former.py > gpurun_out/former.jsonl 2>&1
bash tools/profile_former_tc.sh > gpurun_out/profile_former_tc.log 2>&1
python tools/prof_former_torch.py > gpurun_out/former_torch_profile.txt 2>&1
python tools/run_configs.py > gpurun_out/run_configs.log 2>&1
ls gpurun_out
# summaries on the box (the .ncu-rep captures exceed gpurun's 64 MiB copy-back), then drop the big files
python tools/ncu_summary.py gpurun_out/prof_tc_attn.ncu-rep > gpurun_out/tc_attn_summary.txt 2>&1
python tools/update_profiles.py --round 02 > gpurun_out/update_profiles.log 2>&1
mkdir -p gpurun_out/profiles_r02 && cp profiles/r02_* gpurun_out/profiles_r02/ && cp profiles/k1_traffic.json gpurun_out/profiles_r02/
for f in gpurun_out/*.ncu-rep gpurun_out/*_src.csv; do [ -f "$f" ] && rm -f "$f"; done
du -sh gpurun_out

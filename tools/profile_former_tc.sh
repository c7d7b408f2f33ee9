# Launch list (per-kernel times) of the tensor-core log_prob pipeline on the 16x16-multiplier case, and one
# ncu --set full capture of its attention kernel.
set -x
CMD="python tools/bench_former.py --cases mult16"
$CMD > gpurun_out/former_plain.jsonl 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/former_launches.csv $CMD > gpurun_out/ncu_former_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_tc_attn_mma -s 2 -c 1 -o gpurun_out/prof_tc_attn -f $CMD > gpurun_out/ncu_tc_attn.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_tc_mlp -s 2 -c 1 -o gpurun_out/prof_tc_mlp -f $CMD > gpurun_out/ncu_tc_mlp.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_tc_attn.ncu-rep k_tc_attn_mma > gpurun_out/tc_attn_summary.txt 2>&1
python tools/ncu_summary.py gpurun_out/prof_tc_mlp.ncu-rep k_tc_mlp > gpurun_out/tc_mlp_summary.txt 2>&1

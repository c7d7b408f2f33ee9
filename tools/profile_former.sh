# IsingFormer evidence: throughput lines, then one ncu --set full capture of the sampling kernel
# (2D 16x16, T = 256, B = 4096) and of the log_prob kernel.
set -x
[ -n "$SKIP_BENCH" ] || python tools/bench_former.py > gpurun_out/former.jsonl 2> gpurun_out/former.err
python tools/bench_former.py --cases lat16 > gpurun_out/former_plain.jsonl 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_former -s 1 -c 2 -o gpurun_out/prof_former -f \
    python tools/bench_former.py --cases lat16 > gpurun_out/ncu_former.log 2>&1
tail -1 gpurun_out/ncu_former.log

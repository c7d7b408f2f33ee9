# Round evidence: default bench (plain), launch list of the same command, full ncu of K1 on a slice.
set -x
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
tail -c 3000 gpurun_out/bench_default.json
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_nocpu.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
wc -l gpurun_out/launches.csv
SMALL="python bench.py --instances 296 --sweeps-per-step 100 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
$SMALL > gpurun_out/plain_small.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k1_lattice -s 3 -c 1 -o gpurun_out/prof_k1 -f $SMALL > gpurun_out/ncu_k1.log 2>&1
tail -1 gpurun_out/ncu_k1.log

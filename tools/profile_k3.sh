# K3 evidence on config 4 (16x16 multiplier, 512 semiprimes): the bench.py workload line (GPU and the
# reference CPU path), then one full ncu capture of a 1000-sweep k3_bitcsr launch with source.
set -x
python bench.py --workload cfg4 > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
tail -c 1500 gpurun_out/bench_cfg4.json
python tools/bench_configs.py --configs 4 --steps 1 > gpurun_out/k3_plain.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k3_bitcsr -s 1 -c 1 -o gpurun_out/prof_k3 -f \
    python tools/bench_configs.py --configs 4 --steps 1 > gpurun_out/ncu_k3.log 2>&1
tail -1 gpurun_out/ncu_k3.log
ncu -i gpurun_out/prof_k3.ncu-rep --page source --csv --print-source sass > gpurun_out/k3_src.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/prof_k3.ncu-rep k3_bitcsr > gpurun_out/k3_summary.txt 2>&1
python tools/sass_blocks.py gpurun_out/k3_src.csv 8 >> gpurun_out/k3_summary.txt 2>&1

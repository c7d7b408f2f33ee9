# K2 evidence on config 4 (16x16 multiplier): plain run, then one full ncu capture of k2_csr.
set -x
python tools/bench_configs.py --configs 4 --steps 1 > gpurun_out/k2_plain.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k2_csr -s 1 -c 1 -o gpurun_out/prof_k2 -f \
    python tools/bench_configs.py --configs 4 --steps 1 > gpurun_out/ncu_k2.log 2>&1
tail -1 gpurun_out/ncu_k2.log

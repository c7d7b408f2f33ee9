# K3 evidence on config 4: plain K3 vs K2 rates, then one full ncu capture of k3_bitcsr with source.
set -x
python tools/k3_vs_k2.py > gpurun_out/k3_vs_k2.txt 2>&1
TAPT_K3=1 ncu --set full --clock-control none --import-source on -k regex:k3_bitcsr -s 1 -c 1 -o gpurun_out/prof_k3 -f \
    python tools/bench_configs.py --configs 4 --steps 1 > gpurun_out/ncu_k3.log 2>&1
tail -3 gpurun_out/ncu_k3.log
ncu -i gpurun_out/prof_k3.ncu-rep --page source --csv --print-source sass > gpurun_out/k3_src.csv 2>/dev/null
ncu -i gpurun_out/prof_k3.ncu-rep --page raw --csv > gpurun_out/k3_raw.csv 2>/dev/null

bash tools/k3_ipb.sh
TAPT_K3_IPB=${IPB:-3} ncu --set full --clock-control none --import-source on -k regex:k3_bitcsr -s 1 -c 1 -o gpurun_out/prof_k3 -f \
    python tools/bench_configs.py --configs 4 --steps 1 > gpurun_out/ncu_k3.log 2>&1
tail -2 gpurun_out/ncu_k3.log
ncu -i gpurun_out/prof_k3.ncu-rep --page source --csv --print-source sass > gpurun_out/k3_src.csv 2>/dev/null
ncu -i gpurun_out/prof_k3.ncu-rep --page raw --csv > gpurun_out/k3_raw.csv 2>/dev/null

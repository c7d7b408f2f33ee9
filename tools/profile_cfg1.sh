# K1 on config 1 (2D L=32, 32 slots, 296 seeds): one full ncu capture of a 1000-sweep launch.
python tools/bench_configs.py --configs 1 --steps 1 > gpurun_out/cfg1_plain.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k1_lattice -s 1 -c 1 -o gpurun_out/prof_cfg1 -f \
    python tools/bench_configs.py --configs 1 --steps 1 > gpurun_out/ncu_cfg1.log 2>&1
ncu -i gpurun_out/prof_cfg1.ncu-rep --page source --csv --print-source sass > gpurun_out/cfg1_src.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/prof_cfg1.ncu-rep k1_lattice > gpurun_out/cfg1_summary.txt 2>&1
python tools/sass_blocks.py gpurun_out/cfg1_src.csv 10 >> gpurun_out/cfg1_summary.txt 2>&1

# ncu --set full of the config-4 sweep kernel (K3 by default; TAPT_K3=0 for K2): bash tools/profile_cfg4.sh k3|k2
K=${1:-k3}
set -x
python tools/bench_configs.py --configs 4 --steps 1 > gpurun_out/${K}_plain.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:${K}_ -s 1 -c 1 -o gpurun_out/prof_$K -f \
    python tools/bench_configs.py --configs 4 --steps 1 > gpurun_out/ncu_$K.log 2>&1
tail -1 gpurun_out/ncu_$K.log

# One ncu --set full capture of each config's sweep kernel (configs 1-3: K1; config 4 is
# tools/profile_k3.sh), one step each.  Skipped launches: the energy recomputations after the
# disorder / initialisation (config 3 has two).
for k in ${CONFIGS:-1 2 3}; do
  skip=1; [ $k = 3 ] && skip=2
  python tools/bench_configs.py --configs $k --steps 1 > gpurun_out/plain_cfg$k.json 2>&1 && \
  ncu --set full --clock-control none -k regex:k1_lattice -s $skip -c 1 -o gpurun_out/prof_cfg$k -f \
      python tools/bench_configs.py --configs $k --steps 1 > gpurun_out/ncu_cfg$k.log 2>&1
  python tools/ncu_summary.py gpurun_out/prof_cfg$k.ncu-rep k1_lattice > gpurun_out/cfg${k}_summary.txt 2>&1
done
rm -f gpurun_out/prof_cfg*.ncu-rep

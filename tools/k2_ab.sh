# A/B of library builds on config 4 (K2): bash tools/k2_ab.sh "base m512"  (base = lib/libtapt_b200.so)
for v in $1; do
  LP=paper_2509_23043_b200/lib/variants/libtapt_$v.so; [ "$v" = base ] && LP=paper_2509_23043_b200/lib/libtapt_b200.so
  for rep in 1 2; do
    r=$(TAPT_LIB_PATH=$LP python tools/bench_configs.py --configs 4 2>/dev/null | python -c "import json,sys; print(round(json.loads(sys.stdin.read())['updates_per_s']/1e9,1))")
    echo "build $v -> $r G/s"
  done
done

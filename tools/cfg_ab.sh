# A/B of library builds on configs 1-3: bash tools/cfg_ab.sh "base NAME ..." [configs]
for v in $1; do
  LP=paper_2509_23043_b200/lib/variants/libtapt_$v.so; [ "$v" = base ] && LP=paper_2509_23043_b200/lib/libtapt_b200.so
  echo "build $v: $(TAPT_LIB_PATH=$LP python tools/bench_configs.py --configs ${2:-1,2,3} --steps 2 | python -c 'import json,sys; print([round(json.loads(l)["updates_per_s"]/1e9,1) for l in sys.stdin])')"
done

# A/B of library builds on config 4: bash tools/k3_ab.sh "base NAME ..." (NAME from tools/build_variant.sh)
for v in $1; do
  LP=paper_2509_23043_b200/lib/variants/libtapt_$v.so; [ "$v" = base ] && LP=paper_2509_23043_b200/lib/libtapt_b200.so
  for rep in 1 2; do
    echo "build $v: $(TAPT_LIB_PATH=$LP python tools/bench_configs.py --configs 4 --steps 2 | python -c 'import json,sys; print(round(json.loads(sys.stdin.read())["updates_per_s"]/1e9,1))') G/s"
  done
done

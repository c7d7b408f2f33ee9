# IsingFormer sampling: rows (sequences) per CTA A/B: bash tools/former_rb.sh "4 8 32"
for rb in ${1:-4 8 32}; do
  TAPT_FORMER_RB=$rb python tools/bench_former.py --cases ${2:-lat16,mult16} > gpurun_out/former_rb$rb.jsonl 2>&1
  python - "$rb" <<'PY'
import json, sys
rb = sys.argv[1]
for l in open(f"gpurun_out/former_rb{rb}.jsonl"):
    if l.startswith("{"):
        d = json.loads(l)
        print("rows", rb, d["case"], round(d["sample"]["tokens_per_s"] / 1e6, 2), "Mtok/s, hbm", round(d["sample"]["hbm_frac"], 3))
PY
done

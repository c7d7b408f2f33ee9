python - <<'PY' > gpurun_out/probe_variants.log 2>&1
import os, subprocess, sys
for v in range(8):
    r = subprocess.run([sys.executable, "-c", f"import os; os.environ['TAPT_PROBE_VARIANT']='{v}'; import paper_2509_23043_b200 as T; print({v}, T.probe_decision_rate(1,512,20000)[0]/1e9)"], capture_output=True, text=True)
    print(r.stdout.strip(), r.stderr.strip()[-300:])
PY
cat gpurun_out/probe_variants.log
SMALL="python bench.py --instances 296 --sweeps-per-step 100 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
for v in 0 1 3 5 7; do
  if [ $v = 0 ]; then LP=""; else LP="paper_2509_23043_b200/lib/variants/libtapt_v$v.so"; fi
  TAPT_LIB_PATH=$LP $SMALL > gpurun_out/smallv$v.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/smallv$v.json'));print('variant $v', d['value']/1e9, d['roofline']['kernel_ms_per_launch'])"
done

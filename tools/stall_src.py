"""Warp-stall samples by CUDA source line from `ncu -i REP --page source --csv --print-source cuda`
(one table per source file).  usage: python tools/stall_src.py SRC.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
out, tot = [], 0.0
hdr, fname = None, "?"
for r in rows:
    if r and r[0].startswith("File") or (len(r) == 1 and r[0].endswith((".cu", ".cuh"))):
        fname = r[-1].split("/")[-1]
        continue
    if "Source" in r and "Warp Stall Sampling (All Samples)" in r:
        hdr = r
        isrc, ist, iln = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("#")
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    try:
        v = float(r[ist] or 0)
    except ValueError:
        continue
    tot += v
    out.append((v, fname, r[iln], r[isrc].strip()[:100]))
out.sort(key=lambda x: -x[0])
for v, f, ln, src in out[: int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{100 * v / max(tot, 1):5.1f}%  {f}:{ln}  {src}")

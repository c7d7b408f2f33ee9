"""Top SASS lines by warp-stall samples from `ncu -i REP --page source --csv --print-source sass`.
usage: python tools/stall_lines.py SRC.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = next(k for k, r in enumerate(rows) if "Source" in r)
hdr, data = rows[h], rows[h + 1:]
isrc, ist = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
tot = sum(float(r[ist] or 0) for r in data) or 1.0
top = sorted(range(len(data)), key=lambda k: -float(data[k][ist] or 0))[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]
for k in sorted(top):
    print(f"{100 * float(data[k][ist] or 0) / tot:5.1f}%  {k:5d}  {data[k][isrc][:110]}")

"""Warp-stall samples by SASS opcode from `ncu -i REP --page source --csv --print-source sass`:
which instructions the warps wait on and why.  usage: python tools/stall_ops.py SRC.csv [N]"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if "Source" in r and "# Samples" in r)
isrc = hdr.index("Source")
keys = ["# Samples", "stall_math", "stall_not_selected", "stall_dispatch", "stall_wait", "stall_selected",
        "stall_short_sb", "stall_barrier"]
cols = {k: hdr.index(k) for k in keys if k in hdr}
byop = collections.defaultdict(collections.Counter)
tot = collections.Counter()
for r in rows:
    if len(r) != len(hdr) or r is hdr:
        continue
    m = re.match(r"\s*(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", r[isrc])
    if not m:
        continue
    for k, i in cols.items():
        try:
            v = float(r[i] or 0)
        except ValueError:
            continue
        byop[m.group(1)][k] += v
        tot[k] += v
n = int(sys.argv[2]) if len(sys.argv) > 2 else 12
print("warp-stall samples by opcode (share of all samples; reasons as shares of the opcode's samples)")
print("total samples", int(tot["# Samples"]), {k: f"{100 * v / tot['# Samples']:.1f}%" for k, v in tot.items() if k != "# Samples"})
for op, c in sorted(byop.items(), key=lambda x: -x[1]["# Samples"])[:n]:
    s = c["# Samples"]
    why = ", ".join(f"{k[6:]} {100 * v / s:.0f}%" for k, v in c.most_common() if k != "# Samples" and v > 0.05 * s)
    print(f"  {op:16s} {100 * s / tot['# Samples']:5.1f}%   {why}")

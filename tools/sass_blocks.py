"""Hot basic blocks of a kernel from `ncu -i REP --page source --csv --print-source sass`.

usage: python tools/sass_blocks.py SRC.csv [N]   -- prints the N heaviest runs of equal
execution count (basic blocks) with their share of instructions and stall samples."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = next(k for k, r in enumerate(rows) if "Source" in r)
hdr, data = rows[h], rows[h + 1:]
isrc, iex = hdr.index("Source"), hdr.index("Instructions Executed")
ist = hdr.index("Warp Stall Sampling (All Samples)")
f = lambda x: float(x or 0)
tot = sum(f(r[iex]) for r in data)
stt = sum(f(r[ist]) for r in data) or 1.0
blocks, cur = [], None
for n, r in enumerate(data):
    e = f(r[iex])
    if cur and cur[0] == e:
        cur[2] += 1
        cur[3].append(r[isrc])
        cur[4] += f(r[ist])
    else:
        cur = [e, n, 1, [r[isrc]], f(r[ist])]
        blocks.append(cur)
blocks.sort(key=lambda b: -b[0] * b[2])
print(f"total warp instructions {tot:.4g}")
for e, n, c, srcs, st in blocks[: int(sys.argv[2]) if len(sys.argv) > 2 else 10]:
    ops = collections.Counter(s.split()[1] if s.startswith("@") else s.split()[0] for s in srcs if s.strip())
    print(f"row {n} len {c} x {e:.0f} = {100 * e * c / tot:.1f}% inst, {100 * st / stt:.1f}% stalls ",
          dict(ops.most_common(8)))

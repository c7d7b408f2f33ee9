"""Warp-stall samples of an ncu SASS source page attributed to CUDA source lines, using the line
table of the same build (nvdisasm -gi of the cubin): innermost line and the outermost (kernel-body)
line it was inlined at.
usage: python tools/sass_lines.py SASS.csv CUBIN MANGLED_KERNEL [N]"""
import collections
import csv
import re
import subprocess
import sys

sass_csv, cubin, fn = sys.argv[1:4]
N = int(sys.argv[4]) if len(sys.argv) > 4 else 30
txt = subprocess.run(["nvdisasm", "-gi", "-c", cubin], capture_output=True, text=True).stdout
sec = txt.split(f".text.{fn} ")[1] if f".text.{fn} " in txt else txt.split(f".text.{fn}\n")[1]
sec = sec.split("//---------------------")[0]
loc, cur = {}, ("?", "?")
for line in sec.splitlines():
    m = re.search(r'//## File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?', line)
    if m:
        inner = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
        outer = f"{m.group(3).split('/')[-1]}:{m.group(4)}" if m.group(3) else inner
        cur = (inner, outer)
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", line)
    if m:
        loc[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(sass_csv)))
h = next(k for k, r in enumerate(rows) if "Address" in r and "Source" in r)
hdr, data = rows[h], rows[h + 1:]
ia, ist = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)")
iex = hdr.index("Instructions Executed")
base = int(data[0][ia], 16)
by_in, by_out, ex_out = collections.Counter(), collections.Counter(), collections.Counter()
tot = 0.0
for r in data:
    off = int(r[ia], 16) - base
    v = float(r[ist] or 0)
    inner, outer = loc.get(off, ("?", "?"))
    by_in[inner] += v
    by_out[outer] += v
    ex_out[outer] += float(r[iex] or 0)
    tot += v
print(f"total samples {tot:.0f}")
print("-- by kernel-body line (samples %, executed warp instructions)")
for k, v in by_out.most_common(N):
    print(f"{100 * v / tot:5.1f}%  {ex_out[k]:12.0f}  {k}")
print("-- by innermost line")
for k, v in by_in.most_common(N):
    print(f"{100 * v / tot:5.1f}%  {k}")

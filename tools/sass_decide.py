"""Length of the straight-line SASS blocks that hold >= 32 decisions (VIADDMNMX = the tie-band min)
in a cuobjdump listing: python tools/sass_decide.py FILE.sass"""
import re
import sys

lines = [l for l in open(sys.argv[1]) if re.search(r"/\*[0-9a-f]{4}\*/", l)]
blocks, cur = [], []
for l in lines:
    cur.append(l)
    if re.search(r"\b(BRA|EXIT|BSYNC|RET|BAR|WARPSYNC)\b", l):
        blocks.append(cur)
        cur = []
blocks.append(cur)
for b in blocks:
    k = sum("VIADDMNMX" in l for l in b)
    if k >= 30:
        ops = {}
        for l in b:
            m = re.search(r"\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", l)
            if m:
                ops[m.group(1)] = ops.get(m.group(1), 0) + 1
        top = sorted(ops.items(), key=lambda x: -x[1])[:10]
        print(f"block: {len(b)} instructions, {k} decisions, {len(b) / k:.2f} per decision", top)

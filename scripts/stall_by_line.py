"""Attribute ncu SASS-level warp-stall samples to CUDA source lines (innermost and the
k_peel-level call site) using nvdisasm -gi line tables. Usage:
  stall_by_line.py <ncu source csv (--print-source sass)> <nvdisasm -gi output> <function mangled name>"""
import csv
import re
import sys
from collections import defaultdict

src_csv, sass, fn = sys.argv[1:4]
rows = list(csv.reader(open(src_csv)))
h = rows[1]
iA, iS = h.index("Address"), h.index("Warp Stall Sampling (All Samples)")
iSrc = h.index("Source")
samples = [(int(r[iA], 16), float(r[iS] or 0), r[iSrc]) for r in rows[2:] if len(r) > iS and r[iA].startswith("0x")]
base = min(a for a, _, _ in samples)
lines = open(sass).read().split("\n")
start = next(i for i, l in enumerate(lines) if l.startswith(".text." + fn + ":"))
chain, cur, m = [], [], {}
for l in lines[start + 1:]:
    if l.startswith(".text.") or l.startswith("//----"):
        break
    mm = re.match(r'\s*//## File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?', l)
    if mm:
        cur.append((mm.group(1).split("/")[-1], int(mm.group(2))))
        continue
    mo = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
    if mo:
        if cur:
            chain, cur = cur, []
        m[int(mo.group(1), 16)] = list(chain)
tot = sum(s for _, s, _ in samples)
inner, outer = defaultdict(float), defaultdict(float)
for a, s, txt in samples:
    c = m.get(a - base, [])
    if c:
        inner[c[0]] += s
        outer[c[-1]] += s
print(f"total samples {tot:.0f}")
print("== by k_peel-level line")
for k, v in sorted(outer.items(), key=lambda x: -x[1])[:15]:
    print(f"{v / tot * 100:5.1f}% {k}")
print("== by innermost line")
for k, v in sorted(inner.items(), key=lambda x: -x[1])[:40]:
    print(f"{v / tot * 100:5.1f}% {k}")

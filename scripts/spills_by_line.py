"""Where the local-memory spill instructions (LDL/STL) of a kernel sit: counts per source
line from an `nvdisasm -gi` listing. Usage: spills_by_line.py <listing> <mangled fn substring>"""
import re
import sys
from collections import Counter

dis, fn = sys.argv[1:3]
lines = open(dis).read().split("\n")
start = next(i for i, l in enumerate(lines) if l.startswith(".text.") and fn in l)
cur, cnt, total = None, Counter(), 0
for l in lines[start + 1:]:
    if l.startswith(".text."):
        break
    mm = re.match(r'\s*//## File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?', l)
    if mm:
        cur = (mm.group(1).split("/")[-1], int(mm.group(2)))
        continue
    mo = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s*(.*)", l)
    if mo:
        total += 1
        op = mo.group(2)
        if re.search(r"\b(LDL|STL)\b", op):
            cnt[(cur, "LDL" if "LDL" in op else "STL")] += 1
print("instructions", total, "LDL/STL", sum(cnt.values()))
for (loc, k), c in sorted(cnt.items(), key=lambda kv: (kv[0][0] or ("", 0))):
    print(f"  {loc[0] if loc else '?'}:{loc[1] if loc else 0} {k} x{c}")

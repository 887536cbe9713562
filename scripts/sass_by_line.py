"""Attribute ncu per-SASS-instruction metrics (warp-stall samples and executed warp
instructions) to CUDA source lines via nvdisasm -gi line tables. Usage:
  sass_by_line.py <ncu --page source --csv --print-source sass> <nvdisasm -gi listing> <mangled fn substring> [top]
Prints the innermost source lines and the outermost (kernel-level) call sites ranked by
stall samples, with their share of executed instructions."""
import csv
import re
import sys
from collections import defaultdict

src_csv, dis, fn = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
rows = list(csv.reader(open(src_csv)))
h = rows[1]
iA, iS, iI = h.index("Address"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
iSrc = h.index("Source")
recs = [(int(r[iA], 16), float(r[iS] or 0), float(r[iI] or 0), r[iSrc].strip()) for r in rows[2:]
        if len(r) > iI and r[iA].startswith("0x")]
base = min(a for a, _, _, _ in recs)
lines = open(dis).read().split("\n")
start = next(i for i, l in enumerate(lines) if l.startswith(".text.") and fn in l)
chain, cur, m, sass_txt = [], [], {}, {}
for l in lines[start + 1:]:
    if l.startswith(".text.") or l.startswith("//----"):
        break
    mm = re.match(r'\s*//## File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?', l)
    if mm:
        cur.append((mm.group(1).split("/")[-1], int(mm.group(2))))
        continue
    mo = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s*(.*)", l)
    if mo:
        if cur:
            chain, cur = cur, []
        m[int(mo.group(1), 16)] = list(chain)
        sass_txt[int(mo.group(1), 16)] = mo.group(2)
mism = sum(1 for a, _, _, t in recs if (a - base) in sass_txt and t.split()[0].split(".")[0] not in sass_txt[a - base])
totS = sum(s for _, s, _, _ in recs)
totI = sum(i for _, _, i, _ in recs)
inner, outer = defaultdict(lambda: [0.0, 0.0]), defaultdict(lambda: [0.0, 0.0])
for a, s, i, _ in recs:
    c = m.get(a - base, [])
    if c:
        inner[c[0]][0] += s
        inner[c[0]][1] += i
        outer[c[-1]][0] += s
        outer[c[-1]][1] += i
print(f"total stall samples {totS:.0f}, executed warp instructions {totI:.3e}, opcode mismatches {mism}")
for title, d in (("innermost line", inner), ("kernel-level line", outer)):
    print(f"== by {title}: stall% inst%")
    for k, v in sorted(d.items(), key=lambda x: -x[1][0])[:top]:
        print(f"  {k[0]}:{k[1]:<5} {100 * v[0] / totS:5.1f}% {100 * v[1] / totI:5.1f}%")

"""Summarise a TDG_TRACE dump (level, tasks, probes, ns, K per sub-level) by sub-level size class."""
import sys

rows = [tuple(int(x) for x in l.split()) for l in open(sys.argv[1]) if l.strip()]
classes = [(0, 257, "<=256 (fused)"), (257, 1000, "257-1K"), (1000, 10000, "1K-10K"), (10000, 100000, "10K-100K"),
           (100000, 1 << 20, "100K-1M"), (1 << 20, 1 << 62, ">=1M (sorted)")]
tot_ns = sum(r[3] for r in rows)
print(f"sub-levels {len(rows)} process time {tot_ns/1e6:.1f} ms probes {sum(r[2] for r in rows)/1e9:.2f} G")
print("| tasks per sub-level | sub-levels | probes (G) | time (ms) | share | G probes/s | us per sub-level |")
print("|---|---|---|---|---|---|---|")
for lo, hi, name in classes:
    rs = [r for r in rows if lo <= r[1] < hi]
    if not rs:
        continue
    ns = sum(r[3] for r in rs)
    w = sum(r[2] for r in rs)
    print(f"| {name} | {len(rs)} | {w/1e9:.2f} | {ns/1e6:.1f} | {100*ns/tot_ns:.1f}% | {w/max(ns,1):.1f} | {ns/1e3/len(rs):.1f} |")
top = sorted(rows, key=lambda r: -r[3])[:12]
print("top sub-levels (level, tasks, probes, ms, Gprobes/s):")
for r in top:
    print("  ", r[0], r[1], r[2], round(r[3] / 1e6, 2), round(r[2] / max(r[3], 1), 1))
# fused sub-levels (<= 256 tasks) by probe count W
print("fused sub-levels by probes:")
print("| probes W | sub-levels | time (ms) | us per sub-level |")
print("|---|---|---|---|")
for lo, hi in [(0, 1), (1, 768), (768, 3072), (3072, 12288), (12288, 49152), (49152, 1 << 62)]:
    rs = [r for r in rows if r[1] <= 256 and lo <= r[2] < hi]
    if rs:
        ns = sum(r[3] for r in rs)
        print(f"| {lo}-{hi} | {len(rs)} | {ns/1e6:.2f} | {ns/1e3/len(rs):.1f} |")

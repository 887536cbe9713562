"""Fold gpurun_out/ncu_traffic_C*.csv (scripts/ncu_traffic.sh) into profiles/ncu_traffic.json:
per config and kernel, DRAM bytes per launch, L2 hit rate, L2 atomic / reduction sectors,
instructions, duration, plus the CUDA-source hash of the capture (bench.py uses the file
only while the sources still hash the same)."""
import csv
import glob
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out")
out = {"_doc": "ncu --replay-mode kernel, per decomposition (k_peel: its segments summed; scripts/ncu_traffic.sh); dram_bytes = dram__bytes_read.sum + "
               "dram__bytes_write.sum; atom/red = lts__t_sectors_op_atom/red.sum",
       "src_sha": open(os.path.join(src, "ncu_src_sha.txt")).read().strip()}
for f in sorted(glob.glob(os.path.join(src, "ncu_traffic_C*.csv"))):
    cfg = re.search(r"_C(\d+)\.csv", f).group(1)
    rows = [r for r in csv.reader(ln for ln in open(f) if not ln.startswith("=="))]
    hdr, body = rows[0], rows[1:]
    ix = {k: hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value")}
    per = {}
    for r in body:
        if len(r) < len(hdr):
            continue
        mk = re.search(r"(k_[a-z_0-9]+)", r[ix["Kernel Name"]])
        name = mk.group(1) if mk else r[ix["Kernel Name"]]
        key = (r[ix["ID"]], name)
        v = r[ix["Metric Value"]].replace(",", "")
        try:
            v = float(v)
        except ValueError:
            continue
        unit = r[ix["Metric Unit"]]
        mname = r[ix["Metric Name"]]
        if mname == "gpu__time_duration.sum":
            v = v * {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0,
                     "s": 1e3, "second": 1e3}.get(unit, 1.0)
        if mname.startswith("dram__bytes"):
            v = v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)
        per.setdefault(key, {})[mname] = v
    cf = {}
    for (_, name), d in per.items():
        k = cf.setdefault(name, {"launches": 0})
        k["launches"] += 1
        k["ms"] = k.get("ms", 0) + d.get("gpu__time_duration.sum", 0)
        k["dram_bytes"] = k.get("dram_bytes", 0) + d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
        k["dram_read"] = k.get("dram_read", 0) + d.get("dram__bytes_read.sum", 0)
        k.setdefault("l2_hit_pct_by_launch", []).append(d.get("lts__t_sector_hit_rate.pct"))
        k.setdefault("ms_by_launch", []).append(round(d.get("gpu__time_duration.sum", 0), 3))
        for m_ in ("lts__t_sectors_op_atom.sum", "lts__t_sectors_op_red.sum", "lts__t_requests_op_atom.sum",
                   "lts__t_requests_op_red.sum", "sm__inst_executed.sum"):
            k[m_] = k.get(m_, 0) + d.get(m_, 0)
    # per DECOMPOSITION: k_peel is one logical launch cut into segments (table rebuilds in
    # between); k_support_tab launches once per decomposition
    # (the support pass queues both block geometries; the one the graph does not want exits at once)
    D = max(cf.get("k_support_tab", {}).get("launches", 2) // 2, 1)
    for k in cf.values():
        for m_ in list(k):
            if m_ not in ("launches", "l2_hit_pct_by_launch", "ms_by_launch"):
                k[m_] = k[m_] / D
        w = k["ms_by_launch"]
        k["l2_hit_pct"] = round(sum(a * b for a, b in zip(k["l2_hit_pct_by_launch"], w)) / max(sum(w), 1e-9), 2)
        k["launches_per_decomposition"] = k["launches"] / D
    out[f"C{cfg}"] = cf
dst = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "profiles", "ncu_traffic.json")
json.dump(out, open(dst, "w"), indent=1)
print(json.dumps(out, indent=1))

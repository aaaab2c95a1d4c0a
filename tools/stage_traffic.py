"""Per-stage DRAM traffic and kernel time of one compute() from an ncu CSV
(--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum).
Kernels are assigned to the reference's five StageTimings stages (plus the untimed
assembly) by launch order: each stage starts with a known first kernel.
Usage: python tools/stage_traffic.py launches.csv [out.json]"""
import collections, csv, json, sys

FIRST = [("k_gradient", "gradient"), ("k_compact_crit", "critical"), ("k_compact_crit3", "critical"), ("k_compact_by_dim", "critical"),
         ("k_jump_all", "extrema"), ("k_jump", "extrema"),
         ("k_cp_concat", "assembly"), ("k_succ_table", "reachability"), ("k_scatter_quad_rank", "counting")]
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
per = collections.OrderedDict()  # launch id -> {name, metrics}
for r in rows:
    if "Kernel Name" in r and "Metric Value" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    key = d["ID"]
    e = per.setdefault(key, {"name": d["Kernel Name"].split("(")[0].split("<")[0].split("::")[-1], "m": {}})
    v = float(d["Metric Value"].replace(",", ""))
    unit = d.get("Metric Unit", "")
    scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3,
             "s": 1e3, "byte": 1, "Kbyte": 1e3,
             "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1.0)
    e["m"][d["Metric Name"]] = v * scale
stage = None
out = collections.OrderedDict()
order = [n for _, n in FIRST]
for e in per.values():
    for first, st in FIRST:
        if e["name"] == first and (stage is None or order.index(st) > order.index(stage)):
            stage = st
    if stage is None:
        continue
    s = out.setdefault(stage, {"kernel_ms": 0.0, "dram_bytes": 0.0, "launches": 0, "kernels": {}})
    ms = e["m"].get("gpu__time_duration.sum", 0.0)
    b = e["m"].get("dram__bytes_read.sum", 0.0) + e["m"].get("dram__bytes_write.sum", 0.0)
    s["kernel_ms"] += ms
    s["dram_bytes"] += b
    s["launches"] += 1
    k = s["kernels"].setdefault(e["name"], {"ms": 0.0, "dram_bytes": 0.0, "launches": 0})
    k["ms"] += ms
    k["dram_bytes"] += b
    k["launches"] += 1
for st, s in out.items():
    print(f"{st:14s} {s['kernel_ms']:9.3f} ms  {s['dram_bytes'] / 1e9:8.3f} GB  {s['launches']:4d} launches  "
          f"{s['dram_bytes'] / max(s['kernel_ms'], 1e-9) / 1e6:8.1f} GB/s")
if len(sys.argv) > 2:
    json.dump(out, open(sys.argv[2], "w"), indent=1)

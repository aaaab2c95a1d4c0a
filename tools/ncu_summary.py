"""Aggregate an ncu --csv launch list by kernel name: count, total ms, share."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if "Kernel Name" in r and "Metric Value" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    unit = d.get("Metric Unit", "")
    val = float(d["Metric Value"].replace(",", ""))
    scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(unit, 1e-6)
    name = d["Kernel Name"].split("(")[0]
    agg[name][0] += 1
    agg[name][1] += val * scale
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':60s} {'launches':>8s} {'ms':>10s} {'share':>7s}")
for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k[:60]:60s} {c:8d} {t:10.3f} {100*t/tot:6.1f}%")
print(f"{'TOTAL':60s} {sum(v[0] for v in agg.values()):8d} {tot:10.3f}")

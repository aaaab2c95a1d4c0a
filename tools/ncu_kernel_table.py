"""Per-kernel mean duration / instructions from an `ncu --csv --metrics ...` log (development)."""
import csv, collections, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
agg = collections.defaultdict(list)
for r in rows[1:]:
    agg[(r[ki].split("(")[0][-45:], r[mi])].append(float(r[vi].replace(",", "")))
for (k, mname), v in sorted(agg.items()):
    print(f"{k:45s} {mname:28s} n={len(v):3d} mean={sum(v)/len(v):.4g}")

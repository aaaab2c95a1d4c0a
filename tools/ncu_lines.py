"""Aggregate ncu warp-stall samples per CUDA source line from
`ncu -i rep --page source --csv --print-source cuda,sass` output (stdin or file)."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = None
agg = collections.Counter()
src = {}
cur = None
for r in rows:
    if len(r) > 2 and r[0] == "Line No":
        hdr = r
        si = r.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or not r:
        continue
    if r[0].strip().isdigit():
        cur = int(r[0]); src[cur] = r[1][:110]
    try:
        v = int(r[si])
    except (ValueError, IndexError):
        continue
    if cur is not None:
        agg[cur] += v
tot = sum(agg.values()) or 1
print("total samples", tot)
for ln, v in agg.most_common(top):
    print(f"{v:8d} {100*v/tot:5.1f}%  L{ln:<5d} {src.get(ln,'').strip()}")

"""Aggregate ncu warp-stall samples per CUDA source line, per kernel, from
`ncu -i rep --page source --csv --print-source cuda,sass` output."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
filt = sys.argv[3] if len(sys.argv) > 3 else ""
kern, si, agg, src = None, None, {}, {}
for r in rows:
    if len(r) >= 2 and r[0] == "Function Name":
        kern = r[1]
        agg.setdefault(kern, collections.Counter())
        continue
    if len(r) > 2 and r[0] == "Line No":
        si = r.index("Warp Stall Sampling (All Samples)")
        continue
    if si is None or kern is None or not r or not r[0].strip().isdigit():
        continue
    ln = int(r[0])
    src[(kern, ln)] = r[1][:110]
    try:
        agg[kern][ln] += int(r[si])
    except (ValueError, IndexError):
        pass
for kern, c in agg.items():
    if filt and filt not in kern:
        continue
    tot = sum(c.values()) or 1
    print(f"== {kern[:120]}  samples {tot}")
    for ln, v in c.most_common(top):
        print(f"{v:8d} {100*v/tot:5.1f}%  L{ln:<5d} {src.get((kern, ln), '').strip()}")

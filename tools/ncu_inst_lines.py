"""Per-kernel top CUDA source lines by warp instructions executed, from
`ncu -i rep --page source --csv --print-source cuda,sass` (development)."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
fname, kern, hdr = None, None, None
inst = collections.defaultdict(collections.Counter)
thr = collections.defaultdict(collections.Counter)
src = {}
seen_kernels = []
for r in rows:
    if not r:
        continue
    if r[0] == "File Name":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        kern = r[1].split("(")[0].replace("msc3d_dev::<unnamed>::", "")
        if kern not in seen_kernels:
            seen_kernels.append(kern)
        continue
    if r[0] == "Line No":
        hdr = r
        ii, ti = r.index("Instructions Executed"), r.index("Thread Instructions Executed")
        continue
    if hdr is None or not r[0].strip().isdigit():
        continue
    try:
        a, b = int(r[ii] or 0), int(r[ti] or 0)
    except ValueError:
        continue
    key = (r[1].strip()[:90], int(r[0]))  # (several files share line numbers: key by text too)
    inst[kern][key] += a
    thr[kern][key] += b
    src[key] = r[1].strip()[:90]
for k in seen_kernels:
    tot = sum(inst[k].values()) or 1
    ttot = sum(thr[k].values())
    print(f"== {k}: warp inst {tot:.3e}, thread inst {ttot:.3e}, avg threads {ttot / tot:.1f}")
    for key, v in inst[k].most_common(top):
        print(f"{v:11d} {100 * v / tot:5.1f}% {thr[k][key] / max(v, 1):5.1f}thr line {key[1]:<5d} {src[key]}")

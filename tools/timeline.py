"""Development diagnostic: per-round device timelines of the cooperative BFS and
counting kernels for one compute() on a synthetic BASELINE field."""
import sys
import numpy as np
sys.path.insert(0, "/root/repo")
import paper_2009_03707_b200 as m

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
kind = sys.argv[2] if len(sys.argv) > 2 else "gnoise"
dims = (n, n, n)
ctx = m.Context(0)
ctx.load_values(m.synth(kind, dims), dims)
ctx.compute(m.OPT_SEGMENTATION)
ms = ctx.compute(m.OPT_SEGMENTATION)
print(f"{n}^3 {kind}: stages ms", ["%.2f" % x for x in ms])
for name, first in (("reach_stats", 2), ("count_stats", 1)):
    st = ctx.get(name, np.uint64)
    nr = int(st[0])
    t = st[first:first + min(nr, 255) + 1].astype(np.int64)
    d = np.diff(t) / 1e3
    print(f"{name}: rounds {nr}, total {(t[-1] - t[0]) / 1e3:.0f} us; first rounds us {np.round(d[:12]).tolist()}; "
          f"rounds 12+: n={len(d[12:])} mean {d[12:].mean() if len(d) > 12 else 0:.1f} us sum {d[12:].sum():.0f} us")
try:
    dg = ctx.get("count_diag", np.uint64)
    nr = int(ctx.get("count_stats", np.uint64)[0])
    per = dg[4:4 + 3 * min(nr, 256)].reshape(-1, 3)
    print("count per round: max input len / max parents / frontier size")
    print(per[:40].tolist())
    print("tail rounds 12+: max input len", per[12:, 0].max() if nr > 12 else 0, "max parents", per[12:, 1].max() if nr > 12 else 0,
          "frontier sizes 12+", per[12:40, 2].tolist())
except Exception as e:
    print("no diag", e)
try:
    dg = ctx.get("count_diag", np.uint64)
    ph = dg[900:905].astype(np.float64); it = float(dg[905])
    if it:
        print("tail rounds: warp iterations", int(it), "mean cycles per iteration by phase [gather, alloc, heavy, light, release]",
              np.round(ph / it).tolist())
except Exception as e:
    pass
try:
    dg = ctx.get("count_diag", np.uint64)
    print("slowest tail warp iteration cycles", int(dg[920]), "max T", int(dg[921]), "iterations > 100k cycles", int(dg[922]))
except Exception:
    pass
try:
    dg = ctx.get("count_diag", np.uint64)
    if int(dg[922]):
        print("slow iterations (>100k cycles): mean phase cycles", np.round(dg[930:935].astype(np.float64) / float(dg[922])).tolist())
except Exception:
    pass
if "--all" in sys.argv:
    st = ctx.get("count_stats", np.uint64)
    nr = int(st[0])
    t = st[1:1 + min(nr, 255) + 1].astype(np.int64)
    print("count round us:", np.round(np.diff(t) / 1e3, 1).tolist())
    try:
        print("frontier:", dg[4:4 + 3 * min(nr, 256)].reshape(-1, 3)[:, 2].tolist())
    except Exception as e:
        print(e)

"""Development: per-level time of the reachability BFS (k_reach), from its device clock stamps."""
import sys
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_2009_03707_b200 as m
n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
dims = (n, n, n)
ctx = m.Context(0)
ctx.load_values(m.synth("gnoise", dims), dims)
ctx.compute(m.OPT_SEGMENTATION)
st = ctx.get("reach_stats", np.uint64)
levels = int(st[0])
t = st[2:2 + levels + 1].astype(np.int64)
print("levels", levels, "claims", int(st[1]))
acc = 0.0
for r in range(min(levels, 250)):
    dt = (t[r + 1] - t[r]) / 1e3 if t[r + 1] and t[r] else float("nan")
    acc += dt if dt == dt else 0
    print(f"level {r:3d} {dt:8.1f} us  cumulative {acc / 1e3:6.2f} ms")

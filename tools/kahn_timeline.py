"""Development: per-round timeline of the counting kernel (Kahn's rounds): frontier size
and device time per round (MSC3D_DIAG=1 populates the frontier sizes)."""
import os, sys
os.environ["MSC3D_DIAG"] = "1"
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_2009_03707_b200 as m
n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
dims = (n, n, n)
v = m.synth("gnoise", dims)
ctx = m.Context(0)
ctx.load_values(v, dims)
ctx.compute(m.OPT_SEGMENTATION)
st = ctx.get("count_stats", np.uint64)
dg = ctx.get("count_diag", np.uint64)
rounds = int(st[0])
t = st[1:1 + rounds + 1].astype(np.int64)
print("rounds", rounds)
tot = 0
for r in range(min(rounds, 255)):
    dt = (t[r + 1] - t[r]) / 1e3 if t[r + 1] and t[r] else float("nan")
    light = (int(dg[8 + 3 * r]) - int(t[r])) / 1e3 if dg[8 + 3 * r] else float("nan")
    print(f"round {r:3d} frontier {int(dg[6 + 3 * r]):9d} heavy {int(dg[7 + 3 * r]):6d} "
          f"{dt:8.1f} us (light pass + barrier {light:7.1f} us)")

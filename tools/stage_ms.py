"""Development: mean per-stage ms of compute() (CUDA events inside the pipeline) over a
few runs after warm-up; used for A/B runs of kernel variants selected by env vars."""
import sys
import numpy as np
sys.path.insert(0, "/root/repo")
import paper_2009_03707_b200 as m

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
kind = sys.argv[2] if len(sys.argv) > 2 else "gnoise"
runs = int(sys.argv[3]) if len(sys.argv) > 3 else 5
dims = (n, n, n)
v = m.synth(kind, dims)
ctx = m.Context(0)
ctx.load_values(v, dims)
for _ in range(2):
    ctx.compute(m.OPT_SEGMENTATION)
acc = np.zeros(5)
for _ in range(runs):
    acc += np.array(ctx.compute(m.OPT_SEGMENTATION))
ms = acc / runs
print(f"{kind} {n}^3 stages ms: " + " ".join(f"{x:.2f}" for x in ms) + f"  sum {ms.sum():.2f}", flush=True)

"""Development: per-stage device ms vs the whole compute() (events) on small grids."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
import paper_2009_03707_b200 as m
for n, kind in ((256, "gauss"), (256, "gnoise"), (512, "gauss")):
    dims = (n, n, n)
    c = m.Context(0)
    c.load_values(m.synth(kind, dims), dims)
    for _ in range(3):
        c.compute(m.OPT_SEGMENTATION)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    acc = np.zeros(5)
    K = 5
    torch.cuda.synchronize()
    e0.record()
    for _ in range(K):
        acc += np.array(c.compute(m.OPT_SEGMENTATION))
    e1.record()
    torch.cuda.synchronize()
    print(f"{kind} {n}^3: compute {e0.elapsed_time(e1) / K:.2f} ms, stages " + " ".join(f"{x / K:.2f}" for x in acc),
          flush=True)
    c.close()

"""Development probe: device time of one 1-saddle shard of the post-gradient pipeline
(msc3d_ctx_compute_codes) for G shards, vs the whole -- the multi-GPU step's
per-rank saddle work on one GPU."""
import ctypes as C, sys
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
import paper_2009_03707_b200 as m
n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
dims = (n, n, n)
ctx = m.Context(0)
ctx.load_values(m.synth("gnoise", dims), dims)
ctx.compute(m.OPT_SEGMENTATION)
codes_ptr, ncodes, _ = ctx.array_info("codes")
codes = torch.empty(ncodes, dtype=torch.uint8, device="cuda")
ctx.sync()
import paper_2009_03707_b200.multigpu as mg
src = mg._wrap_device(codes_ptr, ncodes)
codes.copy_(src)
torch.cuda.synchronize()
full = m.Context(0)
m._raise(full._L.msc3d_ctx_bind_codes(full.h, m.Dims(*dims), C.c_void_p(codes.data_ptr())), "bind")
st = (C.c_double * 5)()
for G in (1, 2, 4, 8):
    for r in sorted({0, G // 2, G - 1}):
        best = None
        for rep in range(2):
            m._raise(full._L.msc3d_ctx_compute_codes(full.h, m.OPT_SEGMENTATION, r, G, st), "compute_codes")
            full.sync()
            t = sum(st)
            best = t if best is None else min(best, t)
        print(f"G={G} shard {r}: {best:.1f} ms  stages {[round(x, 1) for x in st]}", flush=True)

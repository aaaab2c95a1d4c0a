"""Development: one msc3d_ctx_compute_host_values call at 512^3 gnoise with MSC3D_DIAG=1
(per-copy ready/start/end on the device clock, widen jobs on the host clock)."""
import ctypes as C, os, sys, time
os.environ["MSC3D_DIAG"] = "1"
import numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2009_03707_b200 as m
n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
dims = (n, n, n)
v = m.synth("gnoise", dims)
ctx = m.Context(0)
hin = torch.from_numpy(v).pin_memory()
ctx.load_values(v, dims)
ctx.compute(m.OPT_SEGMENTATION)
ncp = sum(ctx.scalar(f"c{k}") for k in range(4)); na = ctx.array_info("arc_src")[1]
V = n ** 3; Cu = (n - 1) ** 3
b = {k: torch.empty(sz, dtype=torch.uint8).pin_memory() for k, sz in
     (("cc", ncp * 4), ("ci", ncp), ("as", na * 4), ("ad", na * 4), ("am", na * 8), ("lm", V * 4), ("lx", Cu * 4))}
ho = m.HostOutputs(b["cc"].data_ptr(), ncp * 4, b["ci"].data_ptr(), ncp, b["as"].data_ptr(), b["ad"].data_ptr(),
                   b["am"].data_ptr(), na, b["lm"].data_ptr(), b["lx"].data_ptr(), 0, 0)
for i in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rc = ctx._L.msc3d_ctx_compute_host_values(ctx.h, m.Dims(*dims), m.VALUE_F32, C.c_void_p(hin.data_ptr()),
                                              m.OPT_SEGMENTATION, None, C.byref(ho))
    print(f"call {i}: rc {rc} wall {1e3 * (time.perf_counter() - t0):.1f} ms", file=sys.stderr, flush=True)

"""Development: end-to-end (msc3d_ctx_compute_host_values, host buffers) under D2H delivery
options, interleaved: d2h_threads (host decode threads per narrow array), d2h_dst_first."""
import ctypes as C, sys, time
import numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2009_03707_b200 as m
n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
dims = (n, n, n)
v = m.synth("gnoise", dims)
ctx = m.Context(0)
hin = torch.from_numpy(v).pin_memory()
L = ctx._L
ctx.load_values(v, dims)
ctx.compute(m.OPT_SEGMENTATION)
ncp = sum(ctx.scalar(f"c{k}") for k in range(4)); na = ctx.array_info("arc_src")[1]
V = n ** 3; Cu = (n - 1) ** 3
b = {k: torch.empty(sz, dtype=torch.uint8).pin_memory() for k, sz in
     (("cc", ncp * 4), ("ci", ncp), ("as", na * 4), ("ad", na * 4), ("am", na * 8), ("lm", V * 4), ("lx", Cu * 4))}
ho = m.HostOutputs(b["cc"].data_ptr(), ncp * 4, b["ci"].data_ptr(), ncp, b["as"].data_ptr(), b["ad"].data_ptr(),
                   b["am"].data_ptr(), na, b["lm"].data_ptr(), b["lx"].data_ptr(), 0, 0)
hv = lambda: L.msc3d_ctx_compute_host_values(ctx.h, m.Dims(*dims), m.VALUE_F32, C.c_void_p(hin.data_ptr()),
                                             m.OPT_SEGMENTATION, None, C.byref(ho))
configs = [(0, 0), (8, 0), (4, 0), (0, 1), (8, 1), (12, 0)]
res = {c: [] for c in configs}
ref = None
for rep in range(4):
    for c in configs:
        ctx.set_option("d2h_threads", c[0])
        ctx.set_option("d2h_dst_first", c[1])
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rc = hv()
        torch.cuda.synchronize()
        res[c].append(1e3 * (time.perf_counter() - t0))
        assert rc == 0, rc
        h = hash(bytes(b["am"][: 1 << 20].numpy())) ^ hash(bytes(b["ad"][-(1 << 20):].numpy()))
        ref = h if ref is None else ref
        assert h == ref
for c in configs:
    a = sorted(res[c][1:])
    print(f"d2h_threads {c[0]:2d} dst_first {c[1]}: min {a[0]:.1f} median {a[len(a) // 2]:.1f} ms")

"""Development probe: where the end-to-end time goes (H2D, compute, overlapped D2H)."""
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
def t(f, k=3):
    f(); torch.cuda.synchronize()
    ts = []
    for _ in range(k):
        t0 = time.perf_counter(); f(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    return 1e3 * min(ts)
load = lambda: L.msc3d_ctx_load_values(ctx.h, m.Dims(*dims), m.VALUE_F32, C.c_void_p(hin.data_ptr()))
print("load_values ms", t(load))
print("compute ms", t(lambda: ctx.compute(m.OPT_SEGMENTATION)))
ncp = sum(ctx.scalar(f"c{k}") for k in range(4)); na = ctx.array_info("arc_src")[1]
V = n ** 3; Cu = (n - 1) ** 3
b = {k: torch.empty(sz, dtype=torch.uint8).pin_memory() for k, sz in
     (("cc", ncp * 4), ("ci", ncp), ("as", na * 4), ("ad", na * 4), ("am", na * 8), ("lm", V * 4), ("lx", Cu * 4))}
ho = m.HostOutputs(b["cc"].data_ptr(), ncp * 4, b["ci"].data_ptr(), ncp, b["as"].data_ptr(), b["ad"].data_ptr(),
                   b["am"].data_ptr(), na, b["lm"].data_ptr(), b["lx"].data_ptr(), 0, 0)
for narrow in (1, 0):
    ctx.set_option("d2h_narrow", narrow)
    rcs = []
    ms = t(lambda: rcs.append(L.msc3d_ctx_compute_host(ctx.h, m.OPT_SEGMENTATION, None, C.byref(ho))))
    print(f"compute_host (d2h_narrow {narrow}) ms {ms:.1f} rc {set(rcs)} d2h bytes {ctx.scalar('d2h_bytes') / 1e9:.2f} GB")
    hv = lambda: L.msc3d_ctx_compute_host_values(ctx.h, m.Dims(*dims), m.VALUE_F32, C.c_void_p(hin.data_ptr()),
                                                 m.OPT_SEGMENTATION, None, C.byref(ho))
    print(f"compute_host_values (d2h_narrow {narrow}) ms {t(hv):.1f}")
dev = torch.empty(2 << 30, dtype=torch.uint8, device="cuda")
hb = torch.empty(2 << 30, dtype=torch.uint8).pin_memory()
ms = t(lambda: hb.copy_(dev, non_blocking=True))
print(f"D2H 2 GiB: {ms:.1f} ms = {2 * 1.073741824 / ms * 1e3:.1f} GB/s")
ms = t(lambda: dev.copy_(hb, non_blocking=True))
print(f"H2D 2 GiB: {ms:.1f} ms = {2 * 1.073741824 / ms * 1e3:.1f} GB/s")

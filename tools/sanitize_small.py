"""compute-sanitizer target: the whole pipeline on small grids (device-resident compute
with segmentation, the host-delivery path, the validate audits) -- memcheck / racecheck /
synccheck run this under tools/sanitize.sh."""
import ctypes as C, sys
import numpy as np
sys.path.insert(0, "/root/repo")
import paper_2009_03707_b200 as m

for kind, dims in (("gnoise", (40, 36, 32)), ("noise", (33, 17, 20)), ("gauss", (48, 48, 48))):
    v = m.synth(kind, dims)
    ctx = m.Context(0)
    ctx.load_values(v, dims)
    ctx.compute(m.OPT_SEGMENTATION | m.OPT_VALIDATE)
    ncp = sum(ctx.scalar(f"c{k}") for k in range(4)); na = ctx.array_info("arc_src")[1]
    V = dims[0] * dims[1] * dims[2]; Cu = (dims[0] - 1) * (dims[1] - 1) * (dims[2] - 1)
    buf = {"cc": np.zeros(ncp, np.uint32), "ci": np.zeros(ncp, np.uint8), "as": np.zeros(na, np.uint32),
           "ad": np.zeros(na, np.uint32), "am": np.zeros(na, np.uint64), "lm": np.zeros(V, np.uint32),
           "lx": np.zeros(Cu, np.uint32)}
    p = {k: a.ctypes.data for k, a in buf.items()}
    ho = m.HostOutputs(p["cc"], ncp * 4, p["ci"], ncp, p["as"], p["ad"], p["am"], na, p["lm"], p["lx"], 0, 0)
    rc = ctx._L.msc3d_ctx_compute_host(ctx.h, m.OPT_SEGMENTATION, None, C.byref(ho))
    print(kind, dims, "cps", ncp, "arcs", na, "host rc", rc, flush=True)
    assert rc == 0
print("ok")

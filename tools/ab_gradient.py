"""Development A/B timing of one stage entry point: python tools/ab_gradient.py ROOT KIND N [stage]
(ROOT = a directory holding a paper_2009_03707_b200 package build)."""
import sys
root, kind, n = sys.argv[1], sys.argv[2], int(sys.argv[3])
stage = sys.argv[4] if len(sys.argv) > 4 else "gradient"
sys.path.insert(0, root)
import torch
import paper_2009_03707_b200 as m
dims = (n, n, n)
v = m.synth(kind, dims)
ctx = m.Context(0)
st = torch.cuda.Stream()
ctx._L.msc3d_ctx_set_stream(ctx.h, st.cuda_stream)
ctx.load_values(v, dims)
fn = {"gradient": lambda: ctx.gradient(), "compute": lambda: ctx.compute(m.OPT_SEGMENTATION)}[stage]
for _ in range(2):
    fn()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(5):
    fn()
e1.record(st)
torch.cuda.synchronize()
print(f"{root} {kind} {n}^3 {stage}: {e0.elapsed_time(e1) / 5:.3f} ms")

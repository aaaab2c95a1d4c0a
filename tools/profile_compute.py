"""One compute() on a synthetic grid, bracketed by cudaProfilerStart/Stop, for ncu."""
import ctypes, sys
sys.path.insert(0, "/root/repo")
import paper_2009_03707_b200 as m
n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
kind = sys.argv[2] if len(sys.argv) > 2 else "gnoise"
dims = (n, n, n)
v = m.synth(kind, dims)
ctx = m.Context(0)
ctx.load_values(v, dims)
ctx.compute(m.OPT_SEGMENTATION)  # warm
rt = ctypes.CDLL("libcudart.so.12") if False else None
import torch
torch.cuda.synchronize()
torch.cuda.profiler.start()
ms = ctx.compute(m.OPT_SEGMENTATION)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("stage ms", ms, "launches", ctx.launches())

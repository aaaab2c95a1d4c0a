"""Development: BASELINE config 5 (2048x1024x512 uniform noise, 8.6 G lattice cells) on one
B200 -- does the single-GPU pipeline fit, and what does each stage cost."""
import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np
import torch
import paper_2009_03707_b200 as m

dims = (2048, 1024, 512)
t0 = time.time()
v = m.synth("noise", dims)
print(f"synth {time.time() - t0:.1f}s", flush=True)
ctx = m.Context(0)
ctx.load_values(v, dims)
free0, total = torch.cuda.mem_get_info()
try:
    for i in range(2):
        t0 = time.time()
        ms = ctx.compute(m.OPT_SEGMENTATION)
        print(f"run {i}: wall {time.time() - t0:.2f}s stages ms {[round(x, 1) for x in ms]}", flush=True)
    print("counts", [ctx.scalar(f"c{k}") for k in range(4)], "arcs", ctx.scalar("arcs_min"), ctx.scalar("arcs_ss"),
          ctx.scalar("arcs_max"), "junctions", ctx.scalar("junctions"), flush=True)
except Exception as e:
    print("FAILED:", e, flush=True)
free1, _ = torch.cuda.mem_get_info()
print(f"device memory used by the context: {(free0 - free1) / 1e9:.1f} GB of {total / 1e9:.1f} GB "
      f"(+ inputs {(total - free0) / 1e9:.1f} GB)", flush=True)

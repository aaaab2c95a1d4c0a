"""Development: compute() wall time and device memory at a large grid with the stage
scratch released early (auto above 2^32 cells) or kept (release_transients 0)."""
import sys, time
sys.path.insert(0, "/root/repo")
import torch
import paper_2009_03707_b200 as m
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
kind = sys.argv[2] if len(sys.argv) > 2 else "gauss"
dims = (n, n, n)
v = m.synth(kind, dims)
for rel in (-1, 0):
    ctx = m.Context(0)
    ctx.set_option("release_transients", rel)
    ctx.load_values(v, dims)
    ts = []
    for i in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ms = ctx.compute(m.OPT_SEGMENTATION)
        torch.cuda.synchronize()
        ts.append(1e3 * (time.perf_counter() - t0))
    print(f"release_transients {rel}: compute wall {['%.1f' % t for t in ts]} ms, stages {['%.1f' % x for x in ms]}, "
          f"held {ctx.scalar('device_bytes_held') / 1e9:.1f} GB, peak {ctx.scalar('device_bytes_peak') / 1e9:.1f} GB",
          flush=True)
    del ctx
    torch.cuda.empty_cache()

"""Ad-hoc stage timing (development only): CUDA events on the context's stream."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
import paper_2009_03707_b200 as m

def timeit(fn, stream, iters=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(stream)
    for _ in range(iters):
        fn()
    e.record(stream)
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
kind = sys.argv[2] if len(sys.argv) > 2 else "gnoise"
dims = (n, n, n)
t0 = time.time()
v = m.synth(kind, dims)
print(f"synth {kind} {n}^3: {time.time()-t0:.1f}s", flush=True)
ctx = m.Context(0)
stream = torch.cuda.Stream()
ctx._L.msc3d_ctx_set_stream(ctx.h, stream.cuda_stream)
ctx.load_values(v, dims)
N = m.total_cells(dims)
t = timeit(lambda: ctx.gradient(), stream)
print(f"gradient: {t:.3f} ms  ({(4*n**3 + N)/t/1e6:.0f} GB/s algorithmic)", flush=True)
t = timeit(lambda: ctx.critical(), stream)
print(f"critical (count+compact+sync): {t:.3f} ms  counts {[ctx.scalar(f'c{k}') for k in range(4)]}", flush=True)
t = timeit(lambda: ctx.forest(0), stream)
print(f"forest0: {t:.3f} ms", flush=True)
t = timeit(lambda: ctx.roots(0), stream, iters=2, warm=1)
print(f"roots0 sync-doubling: {t:.3f} ms rounds {ctx.scalar('rounds0')}", flush=True)
t = timeit(lambda: ctx.compute(m.OPT_SEGMENTATION), stream, iters=3, warm=1)
ms = ctx.compute(m.OPT_SEGMENTATION)
print(f"compute: {t:.3f} ms  stages {['%.3f' % x for x in ms]}  levels bfs={ctx.scalar('bfs_levels')} count={ctx.scalar('count_levels')} nodes={ctx.scalar('dag_nodes')} junc={ctx.scalar('junctions')} pool={ctx.scalar('pool_entries')} arcs={ctx.array_info('arc_src')[1]}", flush=True)

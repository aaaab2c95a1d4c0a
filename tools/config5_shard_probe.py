"""Development: per-rank work and device memory of BASELINE config 5 (2048x1024x512
uniform noise, 8.6 G lattice cells, 2-saddle/1-saddle-sharded on 8 B200) emulated on ONE
B200: the gradient once, then for a few shards r of G the post-gradient pipeline a rank
runs on the replicated codes (extrema replicated, reachability + counting on its
1-saddle slice; msc3d_ctx_compute_codes(shard r, G)), with the context's peak device
memory.  The slab gradient of a rank is 1/G of the gradient timed here."""
import ctypes as C
import sys
import time

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
import paper_2009_03707_b200 as m
import paper_2009_03707_b200.multigpu as mg

dims = tuple(int(x) for x in sys.argv[1:4]) if len(sys.argv) >= 4 else (2048, 1024, 512)
kind = sys.argv[4] if len(sys.argv) > 4 else "noise"
G = int(sys.argv[5]) if len(sys.argv) > 5 else 8
shards = [int(x) for x in sys.argv[6].split(",")] if len(sys.argv) > 6 else [0, G // 2, G - 1]
t0 = time.time()
v = m.synth(kind, dims)
print(f"synth {kind} {dims}: {time.time() - t0:.1f}s", flush=True)
total = torch.cuda.mem_get_info()[1]
a = m.Context(0)
a.load_values(v, dims)
del v
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for rep in range(2):
    a.sync()
    t0 = time.time()
    a.gradient()
    a.sync()
    tg = time.time() - t0
print(f"gradient (whole grid, 1 GPU): {tg * 1e3:.1f} ms wall", flush=True)
ptr, n, _ = a.array_info("codes")
codes = torch.empty(n, dtype=torch.uint8, device="cuda")
codes.copy_(mg._wrap_device(ptr, n))
torch.cuda.synchronize()
a.close()
del a
torch.cuda.empty_cache()
free_before = torch.cuda.mem_get_info()[0]
print(f"codes {n / 1e9:.2f} GB resident; free {free_before / 1e9:.1f} of {total / 1e9:.1f} GB", flush=True)
b = m.Context(0)
m._raise(b._L.msc3d_ctx_bind_codes(b.h, m.Dims(*dims), C.c_void_p(codes.data_ptr())), "bind")
st = (C.c_double * 5)()
peak_used = 0
for r in shards:
    try:
        t0 = time.time()
        m._raise(b._L.msc3d_ctx_compute_codes(b.h, m.OPT_SEGMENTATION, r, G, st), "compute_codes")
        b.sync()
        wall = time.time() - t0
    except Exception as e:  # noqa: BLE001
        print(f"shard {r}/{G}: FAILED {e}", flush=True)
        break
    used = b.scalar("device_bytes_held")
    peak_used = max(peak_used, b.scalar("device_bytes_peak"))
    print(f"shard {r}/{G}: stages ms {[round(x, 1) for x in st]} sum {sum(st):.1f}  wall {wall:.2f}s  "
          f"junctions {b.scalar('junctions')} arcs_ss(shard) {b.scalar('arcs_ss')}  "
          f"context holds {used / 1e9:.1f} GB, peak {b.scalar('device_bytes_peak') / 1e9:.1f} GB (+ codes {n / 1e9:.1f} GB)", flush=True)
print(f"peak context memory {peak_used / 1e9:.1f} GB + codes {n / 1e9:.1f} GB of {total / 1e9:.1f} GB", flush=True)

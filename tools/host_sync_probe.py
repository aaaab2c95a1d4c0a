"""Development: host round trips per compute() and the gap between the step's device time
and the sum of its stage times (512^3 gnoise)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
import paper_2009_03707_b200 as m
n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
dims = (n, n, n)
c = m.Context(0)
if len(sys.argv) > 2:
    c.set_option("side_stream", int(sys.argv[2]))
c.load_values(m.synth("gnoise", dims), dims)
for _ in range(2):
    c.compute(m.OPT_SEGMENTATION)
s0, u0 = c.scalar("host_syncs"), c.scalar("host_sync_us")
K = 5
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
acc = np.zeros(5)
torch.cuda.synchronize()
t0 = time.perf_counter()
e0.record()
for _ in range(K):
    acc += np.array(c.compute(m.OPT_SEGMENTATION))
e1.record()
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / K * 1e3
print(f"per compute: wall {wall:.2f} ms, events {e0.elapsed_time(e1) / K:.2f} ms, stage sum {acc.sum() / K:.2f} ms, "
      f"host syncs {(c.scalar('host_syncs') - s0) / K:.1f}, waiting {(c.scalar('host_sync_us') - u0) / K / 1e3:.2f} ms")

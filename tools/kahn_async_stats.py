"""Development: counters of the asynchronous Kahn tail ("kahn_qctl") after one compute()."""
import os
import sys
import numpy as np
os.environ.setdefault("MSC3D_DIAG", "1")
sys.path.insert(0, "/root/repo")
import paper_2009_03707_b200 as m
n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
dims = (n, n, n)
c = m.Context(0)
c.set_option("kahn_async", 1)
c.load_values(m.synth("gnoise", dims), dims)
for i in range(2):
    ms = c.compute(m.OPT_SEGMENTATION)
    q = c.get("kahn_qctl", np.uint64)
    print(f"run {i}: counting {ms[4]:.2f} ms; async kernel {(int(q[42]) - int(q[41])) / 1e3:.1f} us, "
          f"total {int(q[43])} hand-off {int(q[44])} pushed {int(q[16]) - int(q[44])} head {int(q[0])} done {int(q[32])} "
          f"gave-up warps {int(q[40])}; warp iterations {int(q[45])}, lanes busy per iteration "
          f"{int(q[46]) / max(1, int(q[45])):.1f}", flush=True)
    names = ("loads+gather", "pool alloc", "staging", "light merges", "heavy merges", "fence", "release+push",
             "claim+slot+fence")
    it = max(1, int(q[45]))
    print("   cycles per warp iteration: " + ", ".join(f"{nm} {int(q[56 + k]) / it:.0f}" for k, nm in enumerate(names)))
    print(f"   direct merges {int(q[53])} ({int(q[54])} input entries), staging batches {int(q[55])} ({int(q[55]) / it:.2f} per iteration)")

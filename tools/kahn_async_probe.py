"""Development: the asynchronous Kahn tail against the round-based one on small fields,
for several hand-off thresholds (kahn_switch_below)."""
import sys
import numpy as np
sys.path.insert(0, "/root/repo")
import paper_2009_03707_b200 as m

for kind, n in (("gnoise", 16), ("gnoise", 32), ("noise", 24), ("gnoise", 48)):
    dims = (n, n, n)
    v = m.synth(kind, dims)
    ref = m.compute(v, dims, ctx=m.Context(0))
    for sw in (1 << 30, 4096, 64, 1):
        c = m.Context(0)
        c.set_option("kahn_switch_below", sw)
        c.set_option("kahn_async", 1)
        try:
            got = m.compute(v, dims, ctx=c)
            ok = all(np.array_equal(getattr(got, k), getattr(ref, k)) for k in ("arc_src", "arc_dst", "arc_mult"))
            print(kind, n, "switch", sw, "ok" if ok else "MISMATCH", flush=True)
        except Exception as e:  # noqa: BLE001
            print(kind, n, "switch", sw, "FAILED", e, flush=True)
            sys.exit(1)

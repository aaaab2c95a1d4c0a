"""Development: counting-stage ms at 512^3 gnoise for several hand-off thresholds of the
counting kernel (kahn_switch_below), rounds-only vs asynchronous tail."""
import sys
import numpy as np
sys.path.insert(0, "/root/repo")
import paper_2009_03707_b200 as m
n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
kind = sys.argv[2] if len(sys.argv) > 2 else "gnoise"
dims = (n, n, n)
v = m.synth(kind, dims)
for asy in (0, 1):
    for sw in (1 << 16, 1 << 18, 1 << 20, 1 << 21, 1 << 22, 1 << 23):
        c = m.Context(0)
        c.set_option("kahn_async", asy)
        c.set_option("kahn_switch_below", sw)
        c.load_values(v, dims)
        c.compute(m.OPT_SEGMENTATION)
        acc = np.zeros(5)
        for _ in range(3):
            acc += np.array(c.compute(m.OPT_SEGMENTATION))
        print(f"{kind} {n}^3 async {asy} switch 2^{sw.bit_length() - 1}: counting {acc[4] / 3:.2f} ms", flush=True)
        c.close()

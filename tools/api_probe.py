"""Development probe: wall time of the C++ drop-in msc3d::compute() (host ScalarField
of doubles in, host MSComplex out) on a BASELINE field, next to field_hash alone."""
import ctypes as C, sys, time
import numpy as np
sys.path.insert(0, "/root/repo")
import paper_2009_03707_b200 as m
n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
kind = sys.argv[2] if len(sys.argv) > 2 else "gnoise"
v = np.ascontiguousarray(m.synth(kind, (n, n, n)), dtype=np.float32)
L = m.lib()
L.msc3d_api_timed_compute.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int, C.POINTER(C.c_double)]
out = (C.c_double * 8)()
for rep in range(2):
    rc = L.msc3d_api_timed_compute(v.ctypes.data, n, n, n, 1, out)
    print(f"{n}^3 {kind}: rc {rc} compute() {out[0]:.3f} s  cps {int(out[1])} arcs {int(out[2])}  field_hash alone {out[3]:.3f} s", flush=True)

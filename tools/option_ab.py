"""Development: A/B of a context option on the compute() step (stage times, CUDA events),
alternating the settings so clock drift hits both.  Usage: option_ab.py NAME V0 V1 [n] [kind]"""
import sys
sys.path.insert(0, "/root/repo")
import numpy as np
import torch
import paper_2009_03707_b200 as m
name, v0, v1 = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
n = int(sys.argv[4]) if len(sys.argv) > 4 else 512
kind = sys.argv[5] if len(sys.argv) > 5 else "gnoise"
dims = (n, n, n)
v = m.synth(kind, dims)
ctxs = {}
for val in (v0, v1):
    c = m.Context(0)
    c.set_option(name, val)
    c.load_values(v, dims)
    c.compute(m.OPT_SEGMENTATION)
    ctxs[val] = c
ref = {k: ctxs[v0].get(k, np.uint64 if k == "arc_mult" else np.uint32) for k in ("arc_src", "arc_dst", "arc_mult")}
res = {val: [] for val in (v0, v1)}
for it in range(6):
    for val in (v0, v1):
        ms = ctxs[val].compute(m.OPT_SEGMENTATION)
        res[val].append(ms)
for val in (v0, v1):
    a = np.array(res[val][1:])
    med = np.median(a, axis=0)
    print(f"{name}={val}: total {med.sum():.3f} ms  stages {['%.3f' % x for x in med]}", flush=True)
same = all(np.array_equal(ref[k], ctxs[v1].get(k, np.uint64 if k == "arc_mult" else np.uint32)) for k in ref)
print("outputs identical:", same)

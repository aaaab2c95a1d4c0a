"""Development: value distributions of the output arrays (compressibility of the D2H
payload) for one compute() at 512^3 gnoise."""
import sys
import numpy as np
sys.path.insert(0, "/root/repo")
import paper_2009_03707_b200 as m

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
kind = sys.argv[2] if len(sys.argv) > 2 else "gnoise"
dims = (n, n, n)
r = m.compute(m.synth(kind, dims), dims, with_segmentation=True, hash_input=False)
src = r.arc_src.astype(np.int64); dst = r.arc_dst.astype(np.int64); mul = r.arc_mult.astype(np.uint64)
print("arcs", len(src), "sorted src", bool(np.all(np.diff(src) >= 0)))
for lim in (254, 65534, 2**32 - 2):
    print(f"mult > {lim}: {np.count_nonzero(mul > lim)}")
ds = np.diff(src)
print("src delta > 254:", np.count_nonzero(ds > 254), " max", ds.max())
same = ds == 0
dd = np.diff(dst)
print("dst delta within run: <0", np.count_nonzero(dd[same] < 0), " |d|<128", np.count_nonzero(np.abs(dd[same]) < 128),
      " |d|<32768", np.count_nonzero(np.abs(dd[same]) < 32768), " of", same.sum())
nd = dst - src
print("dst - src: |.|<2^15", np.count_nonzero(np.abs(nd) < 2**15), "|.|<2^23", np.count_nonzero(np.abs(nd) < 2**23))
lm = r.labels_min.astype(np.int64)
print("labels_min delta==0 along x", np.count_nonzero(np.diff(lm) == 0) / len(lm))
# signed deltas to the previous entry, whole arrays (candidate i8 / i16 + escapes encodings)
def dstat(name, x):
    d = np.diff(x.astype(np.int64))
    n = max(len(d), 1)
    print(f"{name}: n {len(x)}  |d|<128 {np.count_nonzero(np.abs(d) < 128) / n:.4f}  "
          f"|d|<32768 {np.count_nonzero(np.abs(d) < 32768) / n:.4f}  d==0 {np.count_nonzero(d == 0) / n:.4f}")
dstat("dst (all arcs)", dst)
ncs = [int(np.count_nonzero(src == src))]
dstat("labels_min", lm)
dstat("labels_max", r.labels_max.astype(np.int64))

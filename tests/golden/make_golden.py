"""Generate the committed golden fixtures from the UNMODIFIED reference library.

Run in the build container (where /root/reference exists and oracle/_ref is built):
    make -C oracle ref && python tests/golden/make_golden.py
Each fixture stores the input field and the reference's outputs for every hot-path
stage, so the checkers (and the GPU path) can be pinned without /root/reference.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.pyoracle import Ref  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

CASES = [
    # (name, dims, field maker)
    ("ramp_2x2x2", (2, 2, 2), lambda r, d: _ramp(d)),
    ("ramp_9x4x6", (9, 4, 6), lambda r, d: _ramp(d)),
    ("const_4x3x3", (4, 3, 3), lambda r, d: np.full(int(np.prod(d)), 0.5)),
    ("random_8_s1", (8, 8, 8), lambda r, d: r.generate("white-noise", d, 1)),
    ("random_5x6x7_s2", (5, 6, 7), lambda r, d: r.generate("white-noise", d, 2)),
    ("random_10x9x8_s93", (10, 9, 8), lambda r, d: r.generate("white-noise", d, 93)),
    ("smooth_12_s9", (12, 12, 12), lambda r, d: r.generate("random-smooth", d, 9)),
    ("ties3_9x8x7", (9, 8, 7), lambda r, d: np.random.default_rng(5).integers(0, 3, int(np.prod(d))).astype(np.float64)),
    ("bumps_16", (16, 16, 16), lambda r, d: r.generate("two-bumps", d, 0)),
]


def _ramp(d):
    nx, ny, nz = d
    z, y, x = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    return (x + 2 * y + 4 * z).astype(np.float64).ravel()


def make_case(ref, name, dims, maker):
    v = maker(ref, dims)
    codes = ref.gradient(v, dims)
    crit = ref.critical(codes, dims)
    p0 = ref.forest(codes, dims, 0)
    p3 = ref.forest(codes, dims, 3)
    l0, r0 = ref.roots(p0)
    l3, r3 = ref.roots(p3)
    se = ref.se_arcs(codes, dims, l0, l3)
    marked, ones, twos = ref.mark(codes, dims, crit[1])
    mn = ref.minor(codes, dims, marked, ones, twos)
    cp = ref.count_paths(mn)
    cm = ref.compute(v, dims, with_segmentation=True)
    out = dict(dims=np.array(dims), values=v, codes=codes, p0=p0, p3=p3, l0=l0, l3=l3,
               rounds=np.array([r0, r3]), se_saddle=se[0], se_extremum=se[1], se_mult=se[2],
               marked=marked, one_saddles=ones, two_saddles=twos, junctions=mn["junctions"],
               ss_one=cp[0], ss_two=cp[1], ss_paths=cp[2], cp_cell=cm["cp_cell"],
               cp_index=cm["cp_index"], cp_value=cm["cp_value"], arc_src=cm["arc_src"],
               arc_dst=cm["arc_dst"], arc_mult=cm["arc_mult"], labels_min=cm["labels_min"],
               labels_max=cm["labels_max"], input_hash=np.array([cm["input_hash"]], np.uint64))
    for k in range(4):
        out[f"crit{k}"] = crit[k]
    for k in ("s1_to_j", "j_to_j", "j_to_s2", "s1_to_s2"):
        for j, part in enumerate(("src", "dst", "mult")):
            out[f"{k}.{part}"] = mn[k][j]
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **out)
    return out


def main():
    ref = Ref()
    for name, dims, maker in CASES:
        o = make_case(ref, name, dims, maker)
        print(f"{name}: {len(o['cp_cell'])} critical points, {len(o['arc_src'])} arcs")


if __name__ == "__main__":
    main()

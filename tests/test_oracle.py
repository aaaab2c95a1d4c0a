"""CPU tests (no GPU): the checkers are pinned before they are trusted.

1. oracle64 (our serial restatement, oracle/oracle64.cpp) reproduces the committed
   golden fixtures (tests/golden/*.npz, generated from the unmodified reference by
   tests/golden/make_golden.py) stage by stage.
2. The compiled reference (oracle/_ref) reproduces the reference tests' own known
   answers (proj/tests/test_*.cpp) -- skipped where it was not built.
3. oracle64 == reference on further seeded fields and random minors.
"""
import glob
import os

import numpy as np
import pytest

from oracle.pyoracle import ORC_SO, REF_SO, CheckerError, Oracle64, Ref
from tests.fields import quantized, ramp

GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz")))

need_ref = pytest.mark.skipif(not os.path.exists(REF_SO), reason="oracle/_ref not built")
need_orc = pytest.mark.skipif(not os.path.exists(ORC_SO), reason="oracle/_lib not built")


@pytest.fixture(scope="module")
def orc():
    return Oracle64()


@pytest.fixture(scope="module")
def refc():
    return Ref()


def _minor_from(z):
    mn = {"one_saddles": z["one_saddles"], "junctions": z["junctions"], "two_saddles": z["two_saddles"]}
    for k in ("s1_to_j", "j_to_j", "j_to_s2", "s1_to_s2"):
        mn[k] = (z[f"{k}.src"], z[f"{k}.dst"], z[f"{k}.mult"])
    return mn


def test_golden_fixtures_exist():
    assert len(GOLDEN) >= 8


@need_orc
@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p)[:-4] for p in GOLDEN])
def test_oracle64_matches_golden(orc, path):
    z = np.load(path)
    dims = tuple(int(x) for x in z["dims"])
    v = z["values"]
    codes = orc.gradient(v, dims)
    np.testing.assert_array_equal(codes, z["codes"])
    crit = orc.critical(codes, dims)
    for k in range(4):
        np.testing.assert_array_equal(crit[k], z[f"crit{k}"])
    p0, p3 = orc.forest(codes, dims, 0), orc.forest(codes, dims, 3)
    np.testing.assert_array_equal(p0, z["p0"])
    np.testing.assert_array_equal(p3, z["p3"])
    l0, r0 = orc.roots(p0)
    l3, r3 = orc.roots(p3)
    np.testing.assert_array_equal(l0, z["l0"])
    np.testing.assert_array_equal(l3, z["l3"])
    assert [r0, r3] == z["rounds"].tolist()
    se = orc.se_arcs(codes, dims, l0, l3)
    for got, key in zip(se, ("se_saddle", "se_extremum", "se_mult")):
        np.testing.assert_array_equal(got, z[key])
    marked, ones, twos = orc.mark(codes, dims, crit[1])
    np.testing.assert_array_equal(marked, z["marked"])
    np.testing.assert_array_equal(ones, z["one_saddles"])
    np.testing.assert_array_equal(twos, z["two_saddles"])
    mn = orc.minor(codes, dims, marked, ones, twos)
    want_mn = _minor_from(z)
    np.testing.assert_array_equal(mn["junctions"], want_mn["junctions"])
    for k in ("s1_to_j", "j_to_j", "j_to_s2", "s1_to_s2"):
        for a, b in zip(mn[k], want_mn[k]):
            np.testing.assert_array_equal(a, b)
    cp = orc.count_paths(mn)
    for got, key in zip(cp, ("ss_one", "ss_two", "ss_paths")):
        np.testing.assert_array_equal(got, z[key])
    cm = orc.compute(v, dims)
    for key in ("cp_cell", "cp_index", "cp_value", "arc_src", "arc_dst", "arc_mult", "labels_min", "labels_max"):
        np.testing.assert_array_equal(cm[key], z[key])
    assert cm["input_hash"] == int(z["input_hash"][0])


# ---- the reference tests' known answers, on the compiled reference ----------------------

@need_ref
def test_ref_field_hash_frozen(refc):
    """test_msc.cpp:279-295."""
    assert refc.field_hash(np.array([0.0])) == 0xA8C7F832281A39C5
    assert refc.field_hash(np.array([1.0])) == 0xAAB1693229BA1DB8
    assert refc.field_hash(np.array([0.5, -3.25])) == 0x269A74D4E4AC2BF2


@need_ref
def test_ref_ramp_and_constant(refc):
    """test_gradient.cpp:67-114."""
    for dims in ((2, 2, 2), (16, 16, 16), (9, 4, 6)):
        codes = refc.gradient(ramp(dims), dims)
        assert (codes == 1).sum() == 1 and codes[0] == 1 and (codes == 0).sum() == 0
    codes = refc.gradient(np.full(36, 0.5), (4, 3, 3))
    assert (codes == 1).sum() == 1 and codes[0] == 1


@need_ref
@need_orc
@pytest.mark.parametrize("checker", ["ref", "orc"])
def test_find_roots_chain(refc, orc, checker):
    """test_extrema.cpp:91-107."""
    c = refc if checker == "ref" else orc
    lab, rounds = c.roots(np.array([1, 2, 3, 4, 5, 5]))
    assert rounds == 3 and (lab == 5).all()
    lab, rounds = c.roots(np.array([0, 1, 2, 3]))
    assert rounds == 0


def _labeled_minor(n1, nj, n2):
    return {"one_saddles": np.arange(100, 100 + n1), "junctions": np.arange(500, 500 + nj),
            "two_saddles": np.arange(900, 900 + n2),
            **{k: (np.zeros(0, np.uint32), np.zeros(0, np.uint32), np.zeros(0, np.uint64))
               for k in ("s1_to_j", "j_to_j", "j_to_s2", "s1_to_s2")}}


def _edges(lst):
    if not lst:
        return (np.zeros(0, np.uint32), np.zeros(0, np.uint32), np.zeros(0, np.uint64))
    a = np.array(lst, dtype=object)
    return (np.array([x[0] for x in lst], np.uint32), np.array([x[1] for x in lst], np.uint32),
            np.array([x[2] for x in lst], np.uint64))


HAND_MINORS = [
    # test_path_matrix.cpp:299-332: (n1, nj, n2, edges per kind, expected paths)
    ((1, 0, 1), {"s1_to_s2": [(0, 0, 1)]}, [1]),
    ((1, 1, 1), {"s1_to_j": [(0, 0, 2)], "j_to_s2": [(0, 0, 2)]}, [4]),
    ((1, 2, 1), {"s1_to_j": [(0, 0, 2)], "j_to_j": [(0, 1, 3)], "j_to_s2": [(1, 0, 5)]}, [30]),
    ((1, 2, 1), {"s1_to_j": [(0, 0, 1), (0, 1, 1)], "j_to_s2": [(0, 0, 1), (1, 0, 1)],
                 "s1_to_s2": [(0, 0, 1)]}, [3]),
    ((2, 3, 2), {}, []),
    ((1, 1, 1), {"s1_to_j": [(0, 0, 3)], "s1_to_s2": [(0, 0, 2)]}, [2]),
]


@need_ref
@need_orc
@pytest.mark.parametrize("case", range(len(HAND_MINORS)))
def test_hand_minors(refc, orc, case):
    (n1, nj, n2), edges, want = HAND_MINORS[case]
    mn = _labeled_minor(n1, nj, n2)
    for k, lst in edges.items():
        mn[k] = _edges(lst)
    for c in (refc, orc):
        one, two, paths = c.count_paths(mn)
        assert paths.tolist() == want
        if want:
            assert one.tolist() == [100] and two.tolist() == [900]


@need_ref
@need_orc
def test_count_paths_errors(refc, orc):
    """test_path_matrix.cpp:334-353: cycle -> runtime_error, 64-bit overflow -> overflow_error."""
    cyc = _labeled_minor(1, 2, 1)
    cyc["s1_to_j"] = _edges([(0, 0, 1)])
    cyc["j_to_j"] = _edges([(0, 1, 1), (1, 0, 1)])
    cyc["j_to_s2"] = _edges([(1, 0, 1)])
    big = _labeled_minor(1, 1, 1)
    big["s1_to_j"] = _edges([(0, 0, 1 << 63)])
    big["j_to_s2"] = _edges([(0, 0, 4)])
    sm = _labeled_minor(1, 1, 1)
    sm["s1_to_j"] = _edges([(0, 0, 1 << 63)])
    sm["j_to_s2"] = _edges([(0, 0, 1)])
    sm["s1_to_s2"] = _edges([(0, 0, 1 << 63)])
    # A* overflow at a dead-end junction: no 2-saddle ever sees it (path_matrix.cpp:201-206)
    dead = _labeled_minor(1, 2, 1)
    dead["s1_to_j"] = _edges([(0, 0, 1 << 40)])
    dead["j_to_j"] = _edges([(0, 1, 1 << 40)])
    dead["s1_to_s2"] = _edges([(0, 0, 1)])
    for c in (refc, orc):
        with pytest.raises(CheckerError) as e:
            c.count_paths(cyc)
        assert e.value.kind == "runtime_error"
        for mn in (big, sm, dead):
            with pytest.raises(CheckerError) as e:
                c.count_paths(mn)
            assert e.value.kind == "overflow_error"


def _random_minor(rng):
    """test_path_matrix.cpp:103-123 (index-upward junction edges: a DAG)."""
    n1, nj, n2 = 1 + rng.integers(3), rng.integers(9), 1 + rng.integers(4)
    mn = _labeled_minor(n1, nj, n2)
    e = {k: [] for k in ("s1_to_j", "j_to_j", "j_to_s2", "s1_to_s2")}
    mult = lambda: int(1 + rng.integers(3))
    for i in range(n1):
        e["s1_to_j"] += [(i, j, mult()) for j in range(nj) if rng.integers(100) < 35]
        e["s1_to_s2"] += [(i, j, mult()) for j in range(n2) if rng.integers(100) < 25]
    for i in range(nj):
        e["j_to_j"] += [(i, j, mult()) for j in range(i + 1, nj) if rng.integers(100) < 25]
        e["j_to_s2"] += [(i, j, mult()) for j in range(n2) if rng.integers(100) < 30]
    for k, lst in e.items():
        mn[k] = _edges(lst)
    return mn


@need_ref
@need_orc
def test_random_minors_oracle_equals_reference(refc, orc):
    rng = np.random.default_rng(4242)
    for _ in range(200):
        mn = _random_minor(rng)
        a, b = refc.count_paths(mn), orc.count_paths(mn)
        for x, y in zip(a, b):
            np.testing.assert_array_equal(x, y)


@need_ref
@need_orc
@pytest.mark.parametrize("dims,levels,seed", [((7, 6, 5), 0, 21), ((6, 7, 8), 0, 22), ((9, 8, 7), 3, 1),
                                              ((8, 9, 7), 2, 2), ((11, 5, 6), 5, 3)])
def test_oracle64_equals_reference_compute(refc, orc, dims, levels, seed):
    v = refc.generate("white-noise", dims, seed) if levels == 0 else quantized(dims, levels, seed)
    a, b = refc.compute(v, dims), orc.compute(v, dims)
    for key in ("cp_cell", "cp_index", "cp_value", "arc_src", "arc_dst", "arc_mult", "labels_min", "labels_max"):
        np.testing.assert_array_equal(a[key], b[key])
    assert a["input_hash"] == b["input_hash"]


@need_ref
def test_reference_rejects_wide_grids(refc):
    """grid.cpp:17-20: > 2^32-1 cells is invalid_argument; the reason configs 4-5 need oracle64."""
    assert refc.lib.ref_dims_ok(1024, 1024, 1024) == 1
    assert refc.lib.ref_dims_ok(512, 512, 512) == 0

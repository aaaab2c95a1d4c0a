"""Path-count overflow parity on the device pipeline (path_matrix.cpp:188-219,
SURVEY.md §9.6): the reference throws overflow_error iff some A* entry (1-saddle ->
junction paths) or some final 1-saddle -> 2-saddle count exceeds 2^64 - 1 -- including
junctions that reach no 2-saddle (test_path_matrix.cpp:342-353).

The fields are hand-built gradients with 2^k V-paths (tests/vpaths.py): a chain of k
diamonds ending at terminal 2-saddles ("saddle"), at one dead junction ("dead"), or
branching into two dead junctions ("dead2": at k = 63 the device's dead-path bound
reaches 2^64 while no single A* entry does, so the exact decision runs and must say
"no overflow").  Each case is compared with the unmodified reference on the same
codes through the stage API: mark from the chain's source, then count (dag_count,
the same code path compute() runs), and mark from every critical 1-cell.
"""
import numpy as np
import pytest

import paper_2009_03707_b200 as m
from oracle.pyoracle import CheckerError
from tests.vpaths import diamond_chain

pytestmark = pytest.mark.gpu

CASES = [(10, "saddle", False), (63, "saddle", False), (64, "saddle", True),
         (20, "dead", False), (63, "dead", False), (64, "dead", True), (66, "dead", True),
         (63, "dead2", False), (64, "dead2", True)]


def _ref_count(ref, codes, dims, sources):
    marked, ones, twos = ref.mark(codes, dims, sources)
    try:
        return ref.count_paths(ref.minor(codes, dims, marked, ones, twos))
    except CheckerError as e:
        assert e.kind == "overflow_error", e.kind
        return None


@pytest.mark.parametrize("k,end,overflows", CASES)
def test_vpath_chain_stage_count(ref, k, end, overflows):
    codes, dims, src, _ = diamond_chain(k, end)
    want = _ref_count(ref, codes, dims, np.array([src], np.uint32))
    assert (want is None) == overflows
    with m.Context(0) as c:
        c.load_codes(codes, dims).mark(np.array([src]))
        if overflows:
            with pytest.raises(OverflowError):
                c.count()
            return
        c.count()
        a, b, p = want
        np.testing.assert_array_equal(c.get("ss_one"), a)
        np.testing.assert_array_equal(c.get("ss_two"), b)
        np.testing.assert_array_equal(c.get("ss_paths"), p)
        if end == "saddle":
            assert len(p) == 3 and all(int(x) == 1 << k for x in p)


@pytest.mark.parametrize("k,end,overflows", [c for c in CASES if c[0] >= 63])
def test_vpath_chain_all_sources(ref, k, end, overflows):
    """every critical 1-cell as a source (what compute() does): many more 1-saddles,
    some entering the chain midway"""
    codes, dims, _, _ = diamond_chain(k, end)
    crit1 = ref.critical(codes, dims)[1]
    want = _ref_count(ref, codes, dims, crit1)
    assert (want is None) == overflows
    with m.Context(0) as c:
        c.load_codes(codes, dims).mark(crit1)
        if overflows:
            with pytest.raises(OverflowError):
                c.count()
            return
        c.count()
        for got, w in zip(("ss_one", "ss_two", "ss_paths"), want):
            np.testing.assert_array_equal(c.get(got), w, err_msg=got)


def _device_count_minor(ctx, mn):
    """msc3d_ctx_count_minor (count_paths on a host DagMinor, path_matrix.cpp:188-219)."""
    import ctypes as C
    names = ("s1_to_j", "j_to_j", "j_to_s2", "s1_to_s2")
    keep = []

    def arr(x, dt):
        a = np.ascontiguousarray(x, dtype=dt)
        keep.append(a)
        return a.ctypes.data_as(C.c_void_p)

    srcs = (C.c_void_p * 4)(*[arr(mn[k][0], np.uint32) for k in names])
    dsts = (C.c_void_p * 4)(*[arr(mn[k][1], np.uint32) for k in names])
    mults = (C.c_void_p * 4)(*[arr(mn[k][2], np.uint64) for k in names])
    counts = (C.c_uint64 * 4)(*[len(mn[k][0]) for k in names])
    ones, juncs, twos = (arr(mn[k], np.uint32) for k in ("one_saddles", "junctions", "two_saddles"))
    return ctx._L.msc3d_ctx_count_minor(ctx.h, ones, len(mn["one_saddles"]), juncs, len(mn["junctions"]), twos,
                                        len(mn["two_saddles"]), srcs, dsts, mults, counts, 4)


def _minor(n1, nj, n2, edges):
    mn = {"one_saddles": np.arange(n1) * 2 + 1, "junctions": np.arange(nj) * 2 + 3,
          "two_saddles": np.arange(n2) * 2 + 5}
    for k in ("s1_to_j", "j_to_j", "j_to_s2", "s1_to_s2"):
        e = edges.get(k, [])
        mn[k] = (np.array([x[0] for x in e], np.uint32), np.array([x[1] for x in e], np.uint32),
                 np.array([x[2] for x in e], np.uint64))
    return mn


@pytest.mark.parametrize("batch", [0, 1, 2, 3])
@pytest.mark.parametrize("overflows", [False, True])
def test_exact_dead_junction_check_batched(ref, batch, overflows):
    """Four 1-saddles feed a dead junction chain: their forward total saturates at 2^64,
    so the exact per-source check runs -- in batches of `batch` sources -- and decides
    as the reference does: no overflow while each source's A* entry fits, overflow_error
    when one reaches 2^64 (path_matrix.cpp:188-219, test_path_matrix.cpp:342-353)."""
    big = 1 << 62
    e = {"s1_to_j": [(s, 0, big) for s in range(4)], "j_to_j": [(0, 1, 2 if overflows else 1)],
         "s1_to_s2": [(s, 0, 1) for s in range(4)]}
    if overflows:
        e["s1_to_j"][2] = (2, 0, 1 << 63)
    mn = _minor(4, 2, 1, e)
    try:
        ref.count_paths(mn)
        want_overflow = False
    except CheckerError as err:
        assert err.kind == "overflow_error"
        want_overflow = True
    assert want_overflow == overflows
    with m.Context(0) as c:
        c.set_option("exact_batch_rows", batch)
        rc = _device_count_minor(c, mn)
    assert rc == (m.ERR_OVERFLOW if overflows else m.OK)

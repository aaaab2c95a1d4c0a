"""GPU parity: saddle-graph reachability, path counting and the whole compute().

Fixtures follow proj/tests/test_saddle_graph.cpp, test_path_matrix.cpp and
test_msc.cpp; the checker is the unmodified reference library (oracle/_ref).
"""
import numpy as np
import pytest

import paper_2009_03707_b200 as m
from tests.fields import quantized, ramp, random_field

pytestmark = pytest.mark.gpu


def _codes(ctx, ref, values, dims):
    ctx.load_values(values, dims).gradient()
    return ctx.get("codes")


def _one_saddles(ref, codes, dims):
    return ref.critical(codes, dims)[1]


@pytest.mark.parametrize("dims,seed", [((8, 8, 8), 71), ((8, 8, 8), 72), ((8, 8, 8), 73),
                                       ((6, 7, 5), 71), ((6, 7, 5), 72), ((6, 7, 5), 73)])
def test_mark_reachable_equals_reference(ctx, ref, dims, seed):
    codes = _codes(ctx, ref, random_field(ref, dims, seed), dims)
    src = _one_saddles(ref, codes, dims)
    ctx.mark(src)
    want = ref.mark(codes, dims, src)
    np.testing.assert_array_equal(ctx.get("marked"), want[0])
    np.testing.assert_array_equal(ctx.get("one_saddles"), want[1])
    np.testing.assert_array_equal(ctx.get("two_saddles"), want[2])


@pytest.mark.parametrize("kind", ["gauss", "gnoise", "noise"])
def test_mark_synth(ctx, ref, kind):
    dims = (64, 64, 64)
    codes = _codes(ctx, ref, m.synth(kind, dims), dims)
    src = _one_saddles(ref, codes, dims)
    ctx.mark(None)
    want = ref.mark(codes, dims, src)
    np.testing.assert_array_equal(ctx.get("marked"), want[0])
    np.testing.assert_array_equal(ctx.get("two_saddles"), want[2])


def test_mark_no_saddles(ctx, ref):
    dims = (6, 4, 3)
    _codes(ctx, ref, ramp(dims), dims)
    ctx.mark(np.zeros(0, np.uint32))
    assert ctx.get("marked").sum() == 0
    assert ctx.get("one_saddles").size == 0 and ctx.get("two_saddles").size == 0


def test_mark_rejects_non_saddles(ctx, ref):
    dims = (2, 2, 2)
    _codes(ctx, ref, ramp(dims), dims)
    with pytest.raises(ValueError):
        ctx.mark(np.array([0], np.uint32))  # a vertex
    with pytest.raises(ValueError):
        ctx.mark(np.array([1], np.uint32))  # a paired edge


def _set_pair(codes, dims, lo, hi):
    ex, ey = 2 * dims[0] - 1, 2 * dims[1] - 1
    pack = lambda c: c[0] + ex * (c[1] + ey * c[2])
    axis = 0 if lo[0] != hi[0] else (1 if lo[1] != hi[1] else 2)
    sign = hi[axis] - lo[axis]
    codes[pack(lo)] = m.COFACET_BASE + axis * 2 + (1 if sign > 0 else 0)
    codes[pack(hi)] = m.FACET_BASE + axis * 2 + (1 if -sign > 0 else 0)
    return pack


def test_straight_vpath_fixture(ctx, ref):
    """test_saddle_graph.cpp:35-52,145-171."""
    dims = (2, 2, 2)
    codes = np.full(27, m.CRITICAL, np.uint8)
    pack = _set_pair(codes, dims, (1, 2, 0), (1, 1, 0))
    _set_pair(codes, dims, (1, 0, 1), (1, 1, 1))
    ctx.load_codes(codes, dims)
    e0 = pack((1, 0, 0))
    ctx.mark(np.array([e0], np.uint32))
    want = {e0, pack((1, 1, 0)), pack((1, 2, 0)), pack((1, 2, 1))}
    marked = ctx.get("marked")
    assert set(np.flatnonzero(marked).tolist()) == want
    ctx.count()
    assert ctx.get("ss_one").tolist() == [e0]
    assert ctx.get("ss_two").tolist() == [pack((1, 2, 1))]
    assert ctx.get("ss_paths").tolist() == [1]


def _count_vs_ref(ctx, ref, codes, dims):
    src = _one_saddles(ref, codes, dims)
    marked, ones, twos = ref.mark(codes, dims, src)
    mn = ref.minor(codes, dims, marked, ones, twos)
    want = ref.count_paths(mn)
    ctx.load_codes(codes, dims).mark(src).count()
    got = (ctx.get("ss_one"), ctx.get("ss_two"), ctx.get("ss_paths"))
    for g, w in zip(got, want):
        np.testing.assert_array_equal(g, w)
    return got


@pytest.mark.parametrize("dims,seed", [((8, 8, 8), 91), ((8, 8, 8), 92), ((10, 9, 8), 93),
                                       ((8, 8, 8), 81), ((10, 9, 8), 83), ((9, 8, 7), 94)])
def test_count_paths_random(ctx, ref, dims, seed):
    codes = _codes(ctx, ref, random_field(ref, dims, seed), dims)
    got = _count_vs_ref(ctx, ref, codes, dims)
    assert got[2].size > 0


@pytest.mark.parametrize("kind", ["gauss", "gnoise", "noise"])
def test_count_paths_synth(ctx, ref, kind):
    dims = (48, 48, 48)
    codes = _codes(ctx, ref, m.synth(kind, dims), dims)
    _count_vs_ref(ctx, ref, codes, dims)


def _compute_vs_ref(ctx, ref, values, dims, seg=True):
    got = m.compute(values, dims, with_segmentation=seg, ctx=ctx)
    want = ref.compute(np.asarray(values, dtype=np.float64), dims, with_segmentation=seg)
    np.testing.assert_array_equal(got.cp_cell, want["cp_cell"])
    np.testing.assert_array_equal(got.cp_index.astype(np.int32), want["cp_index"])
    np.testing.assert_array_equal(got.arc_src, want["arc_src"])
    np.testing.assert_array_equal(got.arc_dst, want["arc_dst"])
    np.testing.assert_array_equal(got.arc_mult, want["arc_mult"])
    assert got.input_hash == want["input_hash"]
    if seg:
        np.testing.assert_array_equal(got.labels_min, want["labels_min"])
        np.testing.assert_array_equal(got.labels_max, want["labels_max"])
    assert got.euler() == 1
    return got


@pytest.mark.parametrize("dims,seed", [((8, 8, 8), 101), ((8, 8, 8), 102), ((10, 9, 8), 103),
                                       ((8, 8, 8), 105), ((8, 8, 8), 106), ((9, 8, 7), 107),
                                       ((6, 6, 6), 108)])
def test_compute_random(ctx, ref, dims, seed):
    _compute_vs_ref(ctx, ref, random_field(ref, dims, seed), dims)


def test_compute_ramp(ctx, ref):
    dims = (4, 3, 3)
    got = _compute_vs_ref(ctx, ref, ramp(dims), dims)
    assert got.cp_cell.tolist() == [0] and got.arc_src.size == 0
    assert (got.labels_max == m.NO_LABEL).all()


def test_compute_tie_heavy(ctx, ref):
    for seed in range(3):
        _compute_vs_ref(ctx, ref, quantized((11, 9, 7), 3, seed), (11, 9, 7))


@pytest.mark.parametrize("kind", ["gauss", "gnoise", "noise"])
def test_compute_synth_64(ctx, ref, kind):
    dims = (64, 64, 64)
    got = _compute_vs_ref(ctx, ref, m.synth(kind, dims), dims)
    if kind == "gauss":
        assert [got.count_by_index(k) for k in range(4)] == [134, 461, 356, 28]
        assert got.arc_src.size == 2768 and int(got.arc_mult.max()) == 4


@pytest.mark.parametrize("kind", ["gnoise", "noise"])
def test_bfs_frontier_overflow_retry(ref, kind):
    """A BFS level larger than the frontier buffers is detected and the BFS reruns with
    full-size buffers (stages.cu bfs); the complex is unchanged."""
    dims = (40, 36, 32)
    c = m.Context(0)
    c.set_option("frontier_cap", 64)
    _compute_vs_ref(c, ref, m.synth(kind, dims), dims)
    assert c.scalar("bfs_frontier_retries") == 1
    assert c.scalar("bfs_frontier_cap") == 3 * dims[0] * dims[1] * dims[2]


@pytest.mark.parametrize("kind,dims", [("gnoise", (40, 36, 32)), ("noise", (33, 17, 9)), ("gauss", (48, 40, 36))])
def test_term_rank_words(ref, kind, dims):
    """The 2-saddle rank words in cell order (the walks' terminal lookup above 2^28
    vertices, dag.cu WalkCtx::term_rank) give the same complex as the per-quad map."""
    c = m.Context(0)
    c.set_option("term_rank_words", 1)
    _compute_vs_ref(c, ref, m.synth(kind, dims), dims)
    c.set_option("wide_ids", 1)  # with 64-bit id lists too
    _compute_vs_ref(c, ref, m.synth(kind, dims), dims)


@pytest.mark.parametrize("kind", ["gnoise", "noise"])
def test_side_stream_assembly(ref, kind):
    """Option side_stream: the extremum-side assembly on a second stream gives the same
    complex, device arrays and host deliveries alike."""
    dims = (40, 36, 32)
    c = m.Context(0)
    c.set_option("side_stream", 1)
    for _ in range(2):
        _compute_vs_ref(c, ref, m.synth(kind, dims), dims)


def test_compute_without_segmentation(ctx, ref):
    dims = (8, 8, 8)
    _compute_vs_ref(ctx, ref, random_field(ref, dims, 7), dims, seg=False)


def test_compute_repeatable(ctx, ref):
    dims = (40, 30, 20)
    v = m.synth("gnoise", dims)
    a = m.compute(v, dims, ctx=ctx)
    b = m.compute(v, dims, ctx=ctx)
    for x, y in ((a.arc_src, b.arc_src), (a.arc_dst, b.arc_dst), (a.arc_mult, b.arc_mult),
                 (a.labels_min, b.labels_min)):
        np.testing.assert_array_equal(x, y)


@pytest.mark.parametrize("kind,narrow", [("gnoise", None), ("noise", None),
                                         ("gnoise", {"d2h_narrow_max": 1}),  # escapes (mult + src)
                                         ("noise", {"d2h_narrow_max": 1, "d2h_escape_cap": 200}),
                                         ("noise", {"d2h_narrow_max": 0, "d2h_escape_cap": 3}),  # u64 fallback
                                         ("gnoise", {"d2h_narrow": 0}),  # u64 copies
                                         ("noise", {"side_stream": 1})])  # copies from the side stream
def test_compute_host_outputs(ref, kind, narrow):
    """msc3d_ctx_compute_host: the overlapped host copies (multiplicities as bytes +
    escape list, widened on host threads) equal the reference."""
    import ctypes as C
    ctx = m.Context(0)
    for k, val in (narrow or {}).items():
        ctx.set_option(k, val)
    dims = (40, 36, 32)
    v = m.synth(kind, dims)
    want = ref.compute(v.astype(np.float64), dims, with_segmentation=True)
    ncp, na = len(want["cp_cell"]), len(want["arc_src"])
    V, Cu = dims[0] * dims[1] * dims[2], (dims[0] - 1) * (dims[1] - 1) * (dims[2] - 1)
    buf = {"cp_cell": np.zeros(ncp, np.uint32), "cp_index": np.zeros(ncp, np.uint8),
           "arc_src": np.zeros(na, np.uint32), "arc_dst": np.zeros(na, np.uint32),
           "arc_mult": np.zeros(na, np.uint64), "labels_min": np.zeros(V, np.uint32),
           "labels_max": np.zeros(Cu, np.uint32)}
    ptr = {k: a.ctypes.data for k, a in buf.items()}
    ho = m.HostOutputs(ptr["cp_cell"], ncp * 4, ptr["cp_index"], ncp, ptr["arc_src"], ptr["arc_dst"],
                       ptr["arc_mult"], na, ptr["labels_min"], ptr["labels_max"], 0, 0)
    ctx.load_values(v, dims)
    assert ctx._L.msc3d_ctx_compute_host(ctx.h, m.OPT_SEGMENTATION, None, C.byref(ho)) == 0
    assert ho.n_cp == ncp and ho.n_arcs == na
    for k in ("cp_cell", "arc_src", "arc_dst", "arc_mult", "labels_min", "labels_max"):
        np.testing.assert_array_equal(buf[k], np.asarray(want[k]).astype(buf[k].dtype))
    np.testing.assert_array_equal(buf["cp_index"].astype(np.int32), want["cp_index"])
    # a second delivery (the escape lists now ride with the bytes: sized by this one's)
    for k in ("arc_src", "arc_mult"):
        buf[k][:] = 0
    assert ctx._L.msc3d_ctx_compute_host(ctx.h, m.OPT_SEGMENTATION, None, C.byref(ho)) == 0
    for k in ("arc_src", "arc_dst", "arc_mult"):
        np.testing.assert_array_equal(buf[k], np.asarray(want[k]).astype(buf[k].dtype))
    full = ncp * 5 + na * 16 + (V + Cu) * 4
    if narrow and narrow.get("d2h_narrow") == 0:
        assert ctx.scalar("d2h_bytes") == full
    elif not narrow:
        assert ctx.scalar("d2h_bytes") < full - 6 * na
    # too small an arc buffer is rejected (invalid_argument)
    ho.arc_cap = max(0, na - 1)
    assert ctx._L.msc3d_ctx_compute_host(ctx.h, m.OPT_SEGMENTATION, None, C.byref(ho)) == m.ERR_INVALID


def test_deliver_host(ref):
    """msc3d_ctx_deliver_host: a device-resident compute's outputs delivered to host
    buffers afterwards (the narrow path) equal the reference."""
    import ctypes as C
    ctx = m.Context(0)
    dims = (36, 34, 30)
    v = m.synth("gnoise", dims)
    want = ref.compute(v.astype(np.float64), dims, with_segmentation=True)
    ncp, na = len(want["cp_cell"]), len(want["arc_src"])
    V, Cu = dims[0] * dims[1] * dims[2], (dims[0] - 1) * (dims[1] - 1) * (dims[2] - 1)
    buf = {"cp_cell": np.zeros(ncp, np.uint32), "cp_index": np.zeros(ncp, np.uint8),
           "arc_src": np.zeros(na, np.uint32), "arc_dst": np.zeros(na, np.uint32),
           "arc_mult": np.zeros(na, np.uint64), "labels_min": np.zeros(V, np.uint32),
           "labels_max": np.zeros(Cu, np.uint32)}
    ptr = {k: a.ctypes.data for k, a in buf.items()}
    ho = m.HostOutputs(ptr["cp_cell"], ncp * 4, ptr["cp_index"], ncp, ptr["arc_src"], ptr["arc_dst"],
                       ptr["arc_mult"], na, ptr["labels_min"], ptr["labels_max"], 0, 0)
    assert ctx._L.msc3d_ctx_deliver_host(ctx.h, C.byref(ho)) == m.ERR_STATE  # nothing computed yet
    ctx.load_values(v, dims)
    ctx.compute(m.OPT_SEGMENTATION)
    assert ctx._L.msc3d_ctx_deliver_host(ctx.h, C.byref(ho)) == 0
    assert ho.n_cp == ncp and ho.n_arcs == na
    for k in ("cp_cell", "arc_src", "arc_dst", "arc_mult", "labels_min", "labels_max"):
        np.testing.assert_array_equal(buf[k], np.asarray(want[k]).astype(buf[k].dtype), err_msg=k)


@pytest.mark.parametrize("chunk_kb", ["8", "16", "100000"])
def test_compute_host_values_streamed(ctx, ref, monkeypatch, chunk_kb):
    """msc3d_ctx_compute_host_values: chunked upload overlapped with the gradient, host
    outputs; identical results; non-finite samples rejected (invalid_argument)."""
    import ctypes as C
    monkeypatch.setenv("MSC3D_UPLOAD_CHUNK_KB", chunk_kb)  # 8 KB: 2-plane chunks here
    dims = (33, 29, 70)
    v = m.synth("gnoise", dims)
    want = ref.compute(v.astype(np.float64), dims, with_segmentation=True)
    ncp, na = len(want["cp_cell"]), len(want["arc_src"])
    V, Cu = dims[0] * dims[1] * dims[2], (dims[0] - 1) * (dims[1] - 1) * (dims[2] - 1)
    buf = {"cp_cell": np.zeros(ncp, np.uint32), "cp_index": np.zeros(ncp, np.uint8),
           "arc_src": np.zeros(na, np.uint32), "arc_dst": np.zeros(na, np.uint32),
           "arc_mult": np.zeros(na, np.uint64), "labels_min": np.zeros(V, np.uint32),
           "labels_max": np.zeros(Cu, np.uint32)}
    ptr = {k: a.ctypes.data for k, a in buf.items()}
    ho = m.HostOutputs(ptr["cp_cell"], ncp * 4, ptr["cp_index"], ncp, ptr["arc_src"], ptr["arc_dst"],
                       ptr["arc_mult"], na, ptr["labels_min"], ptr["labels_max"], 0, 0)
    vv = np.ascontiguousarray(v)
    assert ctx._L.msc3d_ctx_compute_host_values(ctx.h, m.Dims(*dims), m.VALUE_F32, vv.ctypes.data,
                                                m.OPT_SEGMENTATION, None, C.byref(ho)) == 0
    for k in ("cp_cell", "arc_src", "arc_dst", "arc_mult", "labels_min", "labels_max"):
        np.testing.assert_array_equal(buf[k], np.asarray(want[k]).astype(buf[k].dtype))
    bad = vv.copy()
    bad[V // 2] = np.nan
    assert ctx._L.msc3d_ctx_compute_host_values(ctx.h, m.Dims(*dims), m.VALUE_F32, bad.ctypes.data,
                                                m.OPT_SEGMENTATION, None, C.byref(ho)) == m.ERR_INVALID

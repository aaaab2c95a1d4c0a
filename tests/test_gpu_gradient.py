"""GPU parity: gradient codes, critical lists, forests, roots, saddle-extremum arcs.

Every case runs the sm_100a kernels through the C ABI (paper_2009_03707_b200 ->
lib/libmsc3d_b200.so) and compares byte-for-byte with the UNMODIFIED reference
library (oracle/_ref) on the same input.  Fixtures follow proj/tests/test_gradient.cpp,
test_extrema.cpp and test_grid.cpp.
"""
import numpy as np
import pytest

import paper_2009_03707_b200 as m
from tests.fields import quantized, ramp, random_field

pytestmark = pytest.mark.gpu

SMALL_RANDOM = [((8, 8, 8), 1), ((8, 8, 8), 2), ((8, 8, 8), 3), ((5, 6, 7), 1), ((5, 6, 7), 2),
                ((5, 6, 7), 3), ((6, 7, 5), 99), ((7, 6, 5), 21), ((2, 2, 2), 5), ((2, 3, 2), 6),
                ((33, 5, 4), 7), ((40, 9, 3), 8)]


def _gpu_codes(ctx, values, dims):
    ctx.load_values(values, dims).gradient()
    return ctx.get("codes")


def _assert_codes(ctx, ref, values, dims):
    got = _gpu_codes(ctx, values, dims)
    want = ref.gradient(np.asarray(values, dtype=np.float64), dims)
    assert got.shape == want.shape
    bad = np.flatnonzero(got != want)
    assert bad.size == 0, f"{bad.size} code mismatches, first at {bad[:8]}: got {got[bad[:8]]} want {want[bad[:8]]}"
    return got


def test_ramp_2x2x2_one_critical(ctx, ref):
    dims = (2, 2, 2)
    codes = _assert_codes(ctx, ref, ramp(dims), dims)
    assert (codes == m.UNSET).sum() == 0
    assert (codes == m.CRITICAL).sum() == 1 and codes[0] == m.CRITICAL


@pytest.mark.parametrize("dims", [(16, 16, 16), (9, 4, 6), (3, 2, 2)])
def test_larger_ramps(ctx, ref, dims):
    codes = _assert_codes(ctx, ref, ramp(dims), dims)
    assert (codes == m.CRITICAL).sum() == 1


def test_constant_field_id_order(ctx, ref):
    dims = (4, 3, 3)
    codes = _assert_codes(ctx, ref, np.full(36, 0.5), dims)
    assert (codes == m.CRITICAL).sum() == 1 and codes[0] == m.CRITICAL


@pytest.mark.parametrize("dims,seed", SMALL_RANDOM)
def test_random_f64(ctx, ref, dims, seed):
    _assert_codes(ctx, ref, random_field(ref, dims, seed), dims)


@pytest.mark.parametrize("levels", [2, 3, 4, 7])
@pytest.mark.parametrize("dims", [(9, 8, 7), (17, 5, 6), (32, 4, 3)])
def test_tie_heavy(ctx, ref, dims, levels):
    """Equal values everywhere: the value-multiset / id-list tie-break path."""
    for seed in range(3):
        _assert_codes(ctx, ref, quantized(dims, levels, seed), dims)


@pytest.mark.parametrize("kind", ["gauss", "gnoise", "noise"])
def test_synthetic_f32_64(ctx, ref, kind):
    dims = (64, 64, 64)
    v = m.synth(kind, dims)
    _assert_codes(ctx, ref, v, dims)


def test_f32_quantized_large(ctx, ref):
    dims = (48, 40, 36)
    v = np.round(m.synth("gnoise", dims) * 16).astype(np.float32)  # heavy ties in f32
    _assert_codes(ctx, ref, v, dims)


def test_nonfinite_rejected(ctx):
    v = np.zeros(8)
    v[3] = np.nan
    with pytest.raises(ValueError):
        ctx.load_values(v, (2, 2, 2))


def _crit(ctx, ref, values, dims):
    ctx.load_values(values, dims).gradient().critical()
    got = [ctx.get(f"crit{k}") for k in range(4)]
    want = ref.critical(ctx.get("codes"), dims)
    for k in range(4):
        np.testing.assert_array_equal(got[k], want[k])
    assert ctx.scalar("euler") == 1
    return got


@pytest.mark.parametrize("dims,seed", SMALL_RANDOM[:6])
def test_critical_lists(ctx, ref, dims, seed):
    _crit(ctx, ref, random_field(ref, dims, seed), dims)


@pytest.mark.parametrize("kind", ["gauss", "gnoise", "noise"])
def test_critical_lists_synth(ctx, ref, kind):
    dims = (64, 64, 64)
    got = _crit(ctx, ref, m.synth(kind, dims), dims)
    if kind == "gauss":  # SURVEY.md §8(d) config 1 counts
        assert [len(x) for x in got] == [134, 461, 356, 28]


def test_critical_lists_multi_tile(ctx, ref):
    dims = (96, 80, 70)  # > 2^20 cells: many look-back tiles
    _crit(ctx, ref, m.synth("noise", dims), dims)


def _forests(ctx, ref, values, dims):
    ctx.load_values(values, dims).gradient()
    codes = ctx.get("codes")
    for dim in (0, 3):
        ctx.forest(dim)
        got = ctx.get("parent0" if dim == 0 else "parent3")
        want = ref.forest(codes, dims, dim)
        np.testing.assert_array_equal(got, want)
        ctx.roots(dim)
        lab = ctx.get("label0" if dim == 0 else "label3")
        wl, wr = ref.roots(want)
        np.testing.assert_array_equal(lab, wl)
        assert ctx.scalar("rounds0" if dim == 0 else "rounds3") == wr
    return codes


@pytest.mark.parametrize("dims,seed", SMALL_RANDOM[:6] + [((64, 64, 64), 0)])
def test_forests_and_roots(ctx, ref, dims, seed):
    v = random_field(ref, dims, seed) if seed else m.synth("gauss", dims)
    _forests(ctx, ref, v, dims)


def test_find_roots_chain(ctx, ref):
    """test_extrema.cpp:91-98: chain {1,2,3,4,5,5} -> 3 rounds, all label 5."""
    ctx.load_codes(np.ones(27, np.uint8), (2, 2, 2))
    ctx.load_parent(0, np.array([1, 2, 3, 4, 5, 5], np.uint32)).roots(0)
    assert ctx.scalar("rounds0") == 3
    assert (ctx.get("label0") == 5).all()
    ctx.load_parent(0, np.array([0, 1, 2, 3], np.uint32)).roots(0)
    assert ctx.scalar("rounds0") == 0


@pytest.mark.parametrize("dims,seed", [((8, 8, 8), 31), ((8, 8, 8), 32), ((8, 8, 8), 33),
                                       ((6, 5, 7), 31), ((6, 5, 7), 32), ((6, 5, 7), 33)])
def test_saddle_extremum_arcs(ctx, ref, dims, seed):
    v = random_field(ref, dims, seed)
    codes = _forests(ctx, ref, v, dims)
    l0, _ = ref.roots(ref.forest(codes, dims, 0))
    l3, _ = ref.roots(ref.forest(codes, dims, 3))
    ctx.se_arcs()
    got = (ctx.get("se_saddle"), ctx.get("se_extremum"), ctx.get("se_mult"))
    want = ref.se_arcs(codes, dims, l0, l3)
    for g, w in zip(got, want):
        np.testing.assert_array_equal(g, w)


def test_se_arcs_synth(ctx, ref):
    dims = (64, 64, 64)
    v = m.synth("gnoise", dims)
    codes = _forests(ctx, ref, v, dims)
    l0, _ = ref.roots(ref.forest(codes, dims, 0))
    l3, _ = ref.roots(ref.forest(codes, dims, 3))
    ctx.se_arcs()
    want = ref.se_arcs(codes, dims, l0, l3)
    for g, w in zip((ctx.get("se_saddle"), ctx.get("se_extremum"), ctx.get("se_mult")), want):
        np.testing.assert_array_equal(g, w)


def test_validate_option_device_audit(ctx):
    """ComputeOptions::validate (msc.cpp:67-70): the device matching audit accepts real
    gradients and rejects tampered ones with runtime_error."""
    dims = (20, 18, 16)
    v = m.synth("gnoise", dims)
    ctx.load_values(v, dims)
    ctx.compute(m.OPT_SEGMENTATION | m.OPT_VALIDATE)
    assert ctx.scalar("validate_violations") == 0
    codes = ctx.get("codes").copy()
    ctx.load_codes(codes, dims)
    assert ctx._L.msc3d_ctx_compute_codes(ctx.h, m.OPT_VALIDATE, 0, 1, None) == m.OK
    paired = np.flatnonzero(codes >= m.FACET_BASE)
    bad = codes.copy()
    bad[paired[len(paired) // 2]] = m.UNSET          # an unassigned cell
    ctx.load_codes(bad, dims)
    assert ctx._L.msc3d_ctx_compute_codes(ctx.h, m.OPT_VALIDATE, 0, 1, None) == m.ERR_RUNTIME
    bad = codes.copy()
    i = paired[len(paired) // 3]
    bad[i] = codes[i] ^ 1                              # pair direction flipped
    ctx.load_codes(bad, dims)                         # a partner that does not pair back
    assert ctx._L.msc3d_ctx_compute_codes(ctx.h, m.OPT_VALIDATE, 0, 1, None) == m.ERR_RUNTIME

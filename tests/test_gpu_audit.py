"""Device audits against the reference:

* validate_gradient (proj/src/gradient.cpp:299-377): matching violations and cells on
  closed V-paths, on the reference's fixtures, tampered codes and a hand-built cycle
  (test_gradient.cpp:67-139 style), compared with the compiled reference;
* boundary_check (proj/src/msc.cpp:149-167): empty on every computed complex (as the
  reference's compute + boundary_check, test_msc.cpp:87-170), and on tampered
  multiplicities (test_msc.cpp:172-207) equal to a direct restatement of the
  reference's loop.
"""
import numpy as np
import pytest

import paper_2009_03707_b200 as m
from tests.fields import quantized, random_field

pytestmark = pytest.mark.gpu


def _fields(ref):
    yield (8, 8, 8), random_field(ref, (8, 8, 8), 1)
    yield (5, 6, 7), random_field(ref, (5, 6, 7), 2)
    yield (9, 8, 7), quantized((9, 8, 7), 3, 4)
    yield (24, 20, 16), m.synth("gnoise", (24, 20, 16)).astype(np.float64)


def _check_report(ctx, ref, codes, dims, max_cells):
    ctx.load_codes(codes, dims)
    got = ctx.validate_gradient(max_cells)
    want = ref.validate_gradient(codes, dims, max_cells)
    assert got["matching_violations"] == want["matching_violations"]
    assert got["cells_in_closed_vpath"] == want["cells_in_closed_vpath"]
    assert got["acyclicity_checked"] == (codes.size <= max_cells)
    return got


@pytest.mark.parametrize("max_cells", [100000, 10 ** 8])
def test_validate_gradient_clean(ctx, ref, max_cells):
    for dims, v in _fields(ref):
        rep = _check_report(ctx, ref, ref.gradient(v, dims), dims, max_cells)
        assert rep["matching_violations"] == 0 and rep["cells_in_closed_vpath"] == 0
        assert not rep["degenerate"]


def test_validate_gradient_tampered(ctx, ref):
    dims = (8, 8, 8)
    codes = ref.gradient(random_field(ref, dims, 3), dims)
    rng = np.random.default_rng(7)
    paired = np.flatnonzero(codes >= m.FACET_BASE)
    bad = codes.copy()
    bad[rng.choice(paired, 25, replace=False)] = m.CRITICAL  # partners no longer point back
    bad[rng.choice(np.flatnonzero(codes == m.CRITICAL), 3, replace=False)] = 0  # unset
    rep = _check_report(ctx, ref, bad, dims, 10 ** 6)
    assert rep["matching_violations"] > 0
    assert len(rep["samples"]) == min(32, rep["matching_violations"])


def test_validate_gradient_closed_vpath(ctx, ref):
    """Four vertices of one face paired around a loop: v00 -> v10 -> v11 -> v01 -> v00."""
    dims = (2, 2, 2)
    ex, ey = 3, 3
    codes = np.full(27, m.CRITICAL, np.uint8)

    def cell(x, y, z):
        return x + ex * (y + ey * z)

    def pair(vx, vy, axis, sign):
        v = cell(2 * vx, 2 * vy, 0)
        e = v + sign * (1 if axis == 0 else ex)
        codes[v] = m.COFACET_BASE + 2 * axis + (sign > 0)
        codes[e] = m.FACET_BASE + 2 * axis + (sign < 0)

    pair(0, 0, 0, +1)
    pair(1, 0, 1, +1)
    pair(1, 1, 0, -1)
    pair(0, 1, 1, -1)
    rep = _check_report(ctx, ref, codes, dims, 10 ** 6)
    assert rep["matching_violations"] == 0 and rep["cells_in_closed_vpath"] == 4


def test_validate_option_rejects_broken_gradient(ctx, ref):
    """compute(validate) throws runtime_error (msc.cpp:67-70) -- here on a 2x2x2 ramp
    whose codes are fine (no throw), then through validate_gradient on broken codes."""
    dims = (6, 5, 4)
    v = random_field(ref, dims, 9)
    ctx.load_values(v, dims)
    ctx.compute(m.OPT_SEGMENTATION | m.OPT_VALIDATE)
    assert ctx.scalar("validate_violations") == 0


def _boundary_restated(cp_index, src, dst, mult):
    """msc.cpp:149-167, restated with dicts (small complexes only)."""
    down = {}
    for a, b, k in zip(src.tolist(), dst.tolist(), mult.tolist()):
        down.setdefault(b, []).append((a, k))
    out = []
    for top in range(len(cp_index)):
        if cp_index[top] < 2:
            continue
        parity = {}
        for mid, k1 in down.get(top, []):
            for low, k2 in down.get(mid, []):
                parity[low] = parity.get(low, 0) ^ (k1 & k2 & 1)
        out += [(top, low) for low in sorted(parity) if parity[low]]
    return np.array(out, dtype=np.uint32).reshape(-1, 2)


def test_boundary_check_clean_and_tampered(ctx, ref):
    for dims, v in _fields(ref):
        got = m.compute(v, dims, with_segmentation=False, ctx=ctx)
        assert ctx.boundary_check().shape == (0, 2)
        want = ref.compute(v, dims, with_segmentation=False, want_text=True)
        assert want["boundary_odd_pairs"] == 0
        idx = got.cp_index.astype(np.uint8)
        rng = np.random.default_rng(dims[0])
        for _ in range(4):
            mult = got.arc_mult.copy()
            flip = rng.choice(len(mult), 3, replace=False)
            mult[flip] += 1
            have = ctx.boundary_check(idx, got.arc_src, got.arc_dst, mult)
            np.testing.assert_array_equal(have, _boundary_restated(idx, got.arc_src, got.arc_dst, mult))

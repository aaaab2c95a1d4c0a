"""GPU parity for two stage-level entry points of the drop-in boundary:

* msc3d_ctx_read_volume against the reference's read_volume (volume.cpp:41-96):
  u8 / u16 / f32 / f64 samples, both byte orders, widening, and the three failure
  kinds (missing file -> IoError, size mismatch / non-finite -> invalid_argument).
  The cases follow proj/tests/test_volume.cpp:36-200.
* msc3d_ctx_minor (build_minor, saddle_graph.cpp:121-217) against the reference's
  build_minor: junction list and the four typed edge lists with multiplicities, on
  the fixtures of proj/tests/test_saddle_graph.cpp:210-235 and synthetic fields.
"""
import numpy as np
import pytest

import paper_2009_03707_b200 as m
from tests.fields import quantized, random_field

pytestmark = pytest.mark.gpu

DTYPES = {"u8": "u1", "u16": "u2", "f32": "f4", "f64": "f8"}


def _device_values(ctx):
    info = ctx.array_info("values")
    return ctx.get("values", np.float64 if info[2] == 8 else np.float32).astype(np.float64)


@pytest.mark.parametrize("dtype", ["u8", "u16", "f32", "f64"])
@pytest.mark.parametrize("big_endian", [False, True])
def test_read_volume_widens_like_reference(tmp_path, ctx, ref, dtype, big_endian):
    dims = (7, 5, 4)
    n = int(np.prod(dims))
    rng = np.random.default_rng(3)
    if dtype in ("u8", "u16"):
        hi = 256 if dtype == "u8" else 65536
        v = rng.integers(0, hi, n)
    else:
        v = rng.standard_normal(n) * 1e3
    path = tmp_path / f"v_{dtype}_{int(big_endian)}.raw"
    np.asarray(v).astype(("<" if not big_endian else ">") + DTYPES[dtype]).tofile(path)
    ctx.read_volume(str(path), dims, dtype, big_endian)
    want = ref.read_volume(str(path), dims, dtype, big_endian)
    np.testing.assert_array_equal(_device_values(ctx), want)


def test_read_volume_known_bytes(tmp_path, ctx):
    """test_volume.cpp:67-110: 0x0102 reads 258 LE / 513 BE; 1.5f = 0x3FC00000."""
    p = tmp_path / "u16.raw"
    p.write_bytes(bytes([0x02, 0x01] * 8))
    ctx.read_volume(str(p), (2, 2, 2), "u16", False)
    np.testing.assert_array_equal(_device_values(ctx), np.full(8, 258.0))
    ctx.read_volume(str(p), (2, 2, 2), "u16", True)
    np.testing.assert_array_equal(_device_values(ctx), np.full(8, 513.0))
    p = tmp_path / "f32.raw"
    p.write_bytes(bytes([0x00, 0x00, 0xC0, 0x3F] * 8))
    ctx.read_volume(str(p), (2, 2, 2), "f32", False)
    np.testing.assert_array_equal(_device_values(ctx), np.full(8, 1.5))


def test_read_volume_failures(tmp_path, ctx, ref):
    dims = (4, 4, 4)
    with pytest.raises(m.IoError):
        ctx.read_volume(str(tmp_path / "missing.raw"), dims, "u8")
    short = tmp_path / "short.raw"
    short.write_bytes(b"\0" * 10)
    with pytest.raises(ValueError):
        ctx.read_volume(str(short), dims, "u8")
    bad = tmp_path / "nan.raw"
    v = np.zeros(64, "<f4")
    v[17] = np.nan
    v.tofile(bad)
    with pytest.raises(ValueError):
        ctx.read_volume(str(bad), dims, "f32")
    inf = tmp_path / "inf.raw"
    w = np.zeros(64, "<f8")
    w[3] = np.inf
    w.tofile(inf)
    with pytest.raises(ValueError):
        ctx.read_volume(str(inf), dims, "f64")
    with pytest.raises(ValueError):
        ctx.read_volume(str(short), dims, "i32")


MINOR_CASES = [
    ("noise", (8, 8, 8), 91),
    ("noise", (8, 8, 8), 92),
    ("noise", (10, 9, 8), 93),
    ("ties", (9, 8, 7), 4),
    ("gnoise", (24, 20, 16), 1),
    ("gauss", (32, 32, 32), 1),
]


@pytest.mark.parametrize("kind,dims,seed", MINOR_CASES)
def test_build_minor_equals_reference(ctx, ref, kind, dims, seed):
    if kind == "noise":
        v = random_field(ref, dims, seed)
    elif kind == "ties":
        v = quantized(dims, 3, seed)
    else:
        v = m.synth(kind, dims, seed=seed).astype(np.float64)
    codes = ref.gradient(v, dims)
    ones = ref.critical(codes, dims)[1]
    ctx.load_codes(codes, dims).mark(ones).minor()
    marked, r1, r2 = ref.mark(codes, dims, ones)
    want = ref.minor(codes, dims, marked, r1, r2)
    np.testing.assert_array_equal(ctx.get("junctions"), want["junctions"])
    for kname in ("s1_to_j", "j_to_j", "j_to_s2", "s1_to_s2"):
        for part, arr in zip(("src", "dst", "mult"), want[kname]):
            np.testing.assert_array_equal(ctx.get(f"{kname}.{part}"), arr, err_msg=f"{kname}.{part}")

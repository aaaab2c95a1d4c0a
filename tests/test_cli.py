"""The msc3d CLI driver (paper_2009_03707_b200/bin/msc3d) -- flags, outputs and exit
codes of the reference CLI (proj/tools/msc3d_cli.cpp:99-166; proj/tests/test_cli.cpp)."""
import os
import subprocess

import numpy as np
import pytest

import paper_2009_03707_b200 as m

BIN = os.path.join(os.path.dirname(m.__file__), "bin", "msc3d")
pytestmark = pytest.mark.skipif(not os.path.exists(BIN), reason="CLI not built")


def run(*args):
    return subprocess.run([BIN, *map(str, args)], capture_output=True, text=True)


def test_usage_and_exit_codes(tmp_path):
    assert run("--help").returncode == 0
    assert run("--bogus").returncode == 1                       # usage error
    assert run("--input", "x.raw").returncode == 1              # missing --dims/--out
    assert run("--dims", "4", "4").returncode == 1              # --dims expects 3 values
    assert run("--input", tmp_path / "missing.raw", "--dims", 4, 4, 4, "--out", tmp_path / "o.json").returncode == 2
    bad = tmp_path / "short.raw"
    bad.write_bytes(b"\0" * 10)                                 # size mismatch -> invalid input
    assert run("--input", bad, "--dims", 4, 4, 4, "--dtype", "f32", "--out", tmp_path / "o.json").returncode == 3


def test_generate_writes_the_baseline_field(tmp_path):
    out = tmp_path / "g.raw"
    r = run("generate", "--kind", "gnoise", "--dims", 12, 10, 8, "--out", out)
    assert r.returncode == 0, r.stderr
    v = np.fromfile(out, dtype="<f4")
    np.testing.assert_array_equal(v, m.synth("gnoise", (12, 10, 8)))
    assert run("generate", "--kind", "ramp", "--dims", 4, 4, 4, "--out", out).returncode == 1


@pytest.mark.gpu
def test_cli_compute_matches_reference(tmp_path, ref):
    dims = (20, 18, 16)
    v = m.synth("gnoise", dims)
    raw = tmp_path / "v.raw"
    v.astype("<f4").tofile(raw)
    pre = tmp_path / "out"
    r = run("--input", raw, "--dims", *dims, "--dtype", "f32", "--format", "csv", "--out", pre,
            "--labels", tmp_path / "lab", "--check")
    assert r.returncode == 0, r.stderr
    want = ref.compute(v.astype(np.float64), dims, with_segmentation=True)
    cps = np.loadtxt(f"{pre}_critical_points.csv", delimiter=",", skiprows=1, ndmin=2)
    np.testing.assert_array_equal(cps[:, 1].astype(np.uint64), np.asarray(want["cp_cell"], dtype=np.uint64))
    arcs = np.loadtxt(f"{pre}_arcs.csv", delimiter=",", skiprows=1, ndmin=2, dtype=np.uint64)
    np.testing.assert_array_equal(arcs[:, 0], np.asarray(want["arc_src"], dtype=np.uint64))
    np.testing.assert_array_equal(arcs[:, 1], np.asarray(want["arc_dst"], dtype=np.uint64))
    np.testing.assert_array_equal(arcs[:, 2], np.asarray(want["arc_mult"], dtype=np.uint64))
    np.testing.assert_array_equal(np.fromfile(tmp_path / "lab_min.raw", dtype="<u4"), want["labels_min"])
    np.testing.assert_array_equal(np.fromfile(tmp_path / "lab_max.raw", dtype="<u4"), want["labels_max"])
    assert "check: euler=1 (ok), mod-2 boundary: 0 odd pairs (ok)" in r.stderr
    r = run("--input", raw, "--dims", *dims, "--dtype", "f32", "--out", tmp_path / "c.json")
    assert r.returncode == 0, r.stderr
    # serialize_json: the same document as the reference's (compared structurally --
    # JSON bytes depend on the json library build)
    import json
    got_doc = json.loads((tmp_path / "c.json").read_text())
    want_doc = json.loads(ref.compute(v.astype(np.float64), dims, with_segmentation=False, dtype="f32",
                                      want_text=True)["json"].decode())
    assert got_doc == want_doc
    assert list(got_doc) == list(want_doc)  # same field order


@pytest.mark.gpu
def test_cli_pinned_f32_ingest_errors(tmp_path):
    """f32 files take the pinned-ingest path (msc3d::compute_volume): a non-finite sample
    is invalid input (exit 3, volume.cpp:89-94 / grid.cpp:86-88), as are u8 / f64 files
    through read_volume, and a big-endian f32 file gives the same complex as the LE one."""
    dims = (12, 10, 8)
    v = m.synth("gnoise", dims)
    bad = v.copy()
    bad[17] = np.nan
    raw = tmp_path / "nan.raw"
    bad.astype("<f4").tofile(raw)
    assert run("--input", raw, "--dims", *dims, "--dtype", "f32", "--out", tmp_path / "o.json").returncode == 3
    le, be = tmp_path / "le.raw", tmp_path / "be.raw"
    v.astype("<f4").tofile(le)
    v.astype(">f4").tofile(be)
    for path, extra in ((le, []), (be, ["--big-endian"])):
        r = run("--input", path, "--dims", *dims, "--dtype", "f32", *extra, "--format", "csv",
                "--out", tmp_path / path.stem)
        assert r.returncode == 0, r.stderr
    assert (tmp_path / "le_arcs.csv").read_bytes() == (tmp_path / "be_arcs.csv").read_bytes()
    assert (tmp_path / "le_critical_points.csv").read_bytes() == (tmp_path / "be_critical_points.csv").read_bytes()


@pytest.mark.gpu
def test_cli_large_complex_matches_reference(tmp_path, ref):
    """A complex large enough that the drop-in compute() takes its parallel host path
    (result vectors >= 64 MB: reserved, huge-page advised, pre-faulted from several
    threads; critical point values from the device): critical points (cell, index,
    doubled coordinates, value), sorted arcs and both label volumes equal the
    unmodified reference's compute() on the same samples (msc.cpp:57-147), and each
    value is the sample at the cell's max vertex (grid.cpp:129-137)."""
    dims = (144, 144, 144)
    v = m.synth("gnoise", dims)
    raw = tmp_path / "v.raw"
    v.astype("<f4").tofile(raw)
    pre = tmp_path / "out"
    r = run("--input", raw, "--dims", *dims, "--dtype", "f32", "--format", "csv", "--out", pre,
            "--labels", tmp_path / "lab")
    assert r.returncode == 0, r.stderr
    r_ = ref.compute(v.astype(np.float64), dims, with_segmentation=True)
    want = type("W", (), {k: r_[k] for k in ("cp_cell", "cp_index", "arc_src", "arc_dst", "arc_mult",
                                             "labels_min", "labels_max")})
    cps = np.loadtxt(f"{pre}_critical_points.csv", delimiter=",", skiprows=1, ndmin=2)
    assert len(cps) > 1_200_000  # >= 64 MB of CriticalPoint records
    np.testing.assert_array_equal(cps[:, 9], r_["cp_value"])
    np.testing.assert_array_equal(cps[:, 0].astype(np.int64), np.arange(len(cps)))
    np.testing.assert_array_equal(cps[:, 1].astype(np.uint64), np.asarray(want.cp_cell, dtype=np.uint64))
    np.testing.assert_array_equal(cps[:, 2].astype(np.uint8), np.asarray(want.cp_index, dtype=np.uint8))
    # doubled coordinates and values, from the cell ids
    nx, ny, nz = dims
    ex, ey = 2 * nx - 1, 2 * ny - 1
    cell = np.asarray(want.cp_cell, dtype=np.int64)
    x, y, z = cell % ex, (cell // ex) % ey, cell // (ex * ey)
    np.testing.assert_array_equal(cps[:, 3:6].astype(np.int64), np.stack([x, y, z], axis=1))
    vol = v.reshape(nz, ny, nx).astype(np.float64)
    best = np.full(len(cell), -np.inf)
    bid = np.full(len(cell), -1, dtype=np.int64)
    for oz in (0, 1):
        for oy in (0, 1):
            for ox in (0, 1):
                ok = ((ox == 0) | (x % 2 == 1)) & ((oy == 0) | (y % 2 == 1)) & ((oz == 0) | (z % 2 == 1))
                vx, vy, vz = x // 2 + ox, y // 2 + oy, z // 2 + oz
                vid = vx + nx * (vy + ny * vz)
                val = np.where(ok, vol[np.minimum(vz, nz - 1), np.minimum(vy, ny - 1), np.minimum(vx, nx - 1)], -np.inf)
                take = ok & ((val > best) | ((val == best) & (vid > bid)))
                best = np.where(take, val, best)
                bid = np.where(take, vid, bid)
    np.testing.assert_array_equal(cps[:, 9], best)
    arcs = np.loadtxt(f"{pre}_arcs.csv", delimiter=",", skiprows=1, ndmin=2, dtype=np.uint64)
    assert arcs.shape[0] * 16 >= 64 << 20
    np.testing.assert_array_equal(arcs[:, 0], np.asarray(want.arc_src, dtype=np.uint64))
    np.testing.assert_array_equal(arcs[:, 1], np.asarray(want.arc_dst, dtype=np.uint64))
    np.testing.assert_array_equal(arcs[:, 2], np.asarray(want.arc_mult, dtype=np.uint64))
    np.testing.assert_array_equal(np.fromfile(tmp_path / "lab_min.raw", dtype="<u4"), want.labels_min)
    np.testing.assert_array_equal(np.fromfile(tmp_path / "lab_max.raw", dtype="<u4"), want.labels_max)

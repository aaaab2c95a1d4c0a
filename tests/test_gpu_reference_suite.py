"""The REFERENCE's own unit tests, compiled unchanged against the B200 drop-in C++ API.

tests/cpp/Makefile compiles /root/reference/proj/tests/{test_grid,test_gradient,
test_extrema,test_saddle_graph,test_path_matrix,test_msc}.cpp (with a doctest shim,
tests/cpp/doctest.h) against include/msc3d/*.hpp and links lib/libmsc3d_b200.so, so
every assign_gradient / extract_critical_cells / find_roots / mark_reachable /
build_minor / count_paths / sp_multiply / compute call in those tests runs on the GPU.
The binary is built in the build container (it needs the reference sources) and
travels to the GPU box; the test is skipped where it was not built.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "_bin", "msc3d_ref_unit_tests")

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not os.path.exists(BIN), reason="reference unit tests not built (make -C tests/cpp)")
def test_reference_unit_suite_on_gpu():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=900)
    tail = (r.stdout[-4000:] + "\n" + r.stderr[-4000:])
    assert r.returncode == 0, tail
    assert "| 0 failed" in r.stdout, tail

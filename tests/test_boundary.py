"""CPU tests of the drop-in boundary: the C-ABI library loads, exports every function
include/msc3d_cuda.h declares, rejects bad dims like GridDims, and fails loudly
(no CPU fallback) when there is no GPU."""
import ctypes as C
import os
import re

import pytest

import paper_2009_03707_b200 as m

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "msc3d_cuda.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(msc3d_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_pipeline():
    names = declared_functions()
    for must in ("msc3d_ctx_gradient", "msc3d_ctx_critical", "msc3d_ctx_forest", "msc3d_ctx_roots",
                 "msc3d_ctx_se_arcs", "msc3d_ctx_mark", "msc3d_ctx_minor", "msc3d_ctx_count",
                 "msc3d_ctx_compute", "msc3d_ctx_read_volume", "msc3d_ctx_load_values"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(m.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_python_mirror_binds_every_symbol():
    L = m.lib()
    for n in declared_functions():
        assert getattr(L, n).restype is not None or n.endswith("_destroy"), n


def test_check_dims_matches_griddims():
    m.check_dims((2, 2, 2))
    m.check_dims((512, 512, 512))
    with pytest.raises(ValueError):
        m.check_dims((1, 5, 5))
    with pytest.raises(ValueError):
        m.check_dims((4, 0, 4))
    with pytest.raises(ValueError):
        m.check_dims((1024, 1024, 1024))  # > 2^32-1 cells (grid.cpp:17-20)
    m.check_dims((1024, 1024, 1024), allow_wide=True)  # the B200 build widens ids
    assert m.id_dtype((512, 512, 512)).__name__ == "uint32"
    assert m.id_dtype((1024, 1024, 1024)).__name__ == "uint64"


def test_field_hash_frozen_values():
    """test_msc.cpp:279-289, host-side FNV-1a of the widened samples."""
    import numpy as np
    L = m.lib()
    for vals, want in (([0.0], 0xA8C7F832281A39C5), ([1.0], 0xAAB1693229BA1DB8),
                       ([0.5, -3.25], 0x269A74D4E4AC2BF2)):
        a = np.array(vals, dtype=np.float64)
        assert L.msc3d_field_hash_f64(a.ctypes.data_as(C.c_void_p), a.size) == want
        f = a.astype(np.float32)
        assert L.msc3d_field_hash_f32(f.ctypes.data_as(C.c_void_p), f.size) == want


def test_no_silent_cpu_fallback():
    """Without a device the context refuses to exist; nothing computes on the host."""
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        m.Context(0)

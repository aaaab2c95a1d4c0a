"""msc3d on B200: Python host mirror of the reference's public API.

The reference (``/root/reference/proj/include/msc3d/*.hpp``) is a C++ library; its
drop-in replacement is the C++ layer in ``csrc/msc3d_api.cpp`` over the C ABI in
``include/msc3d_cuda.h``.  This module binds the same C ABI with ctypes and mirrors
the reference's entry points (same names, same argument meaning, same error
behaviour: ``ValueError`` for ``std::invalid_argument``, ``OverflowError`` for
``std::overflow_error``, ``RuntimeError`` for ``std::runtime_error``) so that the
parity tests read like the reference's own tests.

There is no CPU fallback: every function runs the hand-written sm_100a kernels in
``lib/libmsc3d_b200.so`` and raises if that library or a GPU is missing.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libmsc3d_b200.so")
SYNTH_PATH = os.path.join(HERE, "lib", "libmsc3d_synth.so")

OK, ERR_INVALID, ERR_OVERFLOW, ERR_RUNTIME, ERR_CUDA, ERR_NOMEM, ERR_IO, ERR_STATE = range(8)
VALUE_F32, VALUE_F64 = 0, 1
OPT_SEGMENTATION, OPT_VALIDATE = 1, 2
NO_LABEL = 0xFFFFFFFF

# pair codes (gradient.hpp:29-41)
UNSET, CRITICAL, FACET_BASE, COFACET_BASE = 0, 1, 2, 8


class Dims(C.Structure):
    _fields_ = [("nx", C.c_int64), ("ny", C.c_int64), ("nz", C.c_int64)]


class HostOutputs(C.Structure):
    """msc3d_host_outputs (include/msc3d_cuda.h): host buffers for msc3d_ctx_compute_host."""
    _fields_ = [("cp_cell", C.c_void_p), ("cp_cell_cap", C.c_uint64), ("cp_index", C.c_void_p),
                ("cp_index_cap", C.c_uint64), ("arc_src", C.c_void_p), ("arc_dst", C.c_void_p),
                ("arc_mult", C.c_void_p), ("arc_cap", C.c_uint64), ("labels_min", C.c_void_p),
                ("labels_max", C.c_void_p), ("n_cp", C.c_uint64), ("n_arcs", C.c_uint64)]


# msc3d_host_transport (include/msc3d_cuda.h): allgather(user, send, recv, bytes) -> 0 ok
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64)


class HostTransport(C.Structure):
    _fields_ = [("user", C.c_void_p), ("allgather", ALLGATHER_FN)]


class IoError(RuntimeError):
    pass


_lib = None


def lib():
    """Load the CUDA library (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run __graft_entry__.build() or make -C paper_2009_03707_b200")
    L = C.CDLL(LIB_PATH)
    vp, u64, i64, i32 = C.c_void_p, C.c_uint64, C.c_int64, C.c_int
    sig = {
        "msc3d_status_string": (C.c_char_p, [i32]),
        "msc3d_check_dims": (i32, [Dims, i32]),
        "msc3d_id_width": (i32, [Dims]),
        "msc3d_total_cells": (u64, [Dims]),
        "msc3d_ctx_create": (i32, [C.POINTER(vp), i32]),
        "msc3d_ctx_destroy": (None, [vp]),
        "msc3d_ctx_set_stream": (i32, [vp, vp]),
        "msc3d_ctx_stream": (vp, [vp]),
        "msc3d_ctx_sync": (i32, [vp]),
        "msc3d_ctx_launches": (u64, [vp]),
        "msc3d_ctx_array": (i32, [vp, C.c_char_p, C.POINTER(vp), C.POINTER(u64), C.POINTER(i32)]),
        "msc3d_ctx_download": (i32, [vp, C.c_char_p, vp, u64]),
        "msc3d_ctx_scalar": (i32, [vp, C.c_char_p, C.POINTER(i64)]),
        "msc3d_ctx_set_option": (i32, [vp, C.c_char_p, i64]),
        "msc3d_ctx_load_values": (i32, [vp, Dims, i32, vp]),
        "msc3d_ctx_bind_values": (i32, [vp, Dims, i32, vp]),
        "msc3d_ctx_read_volume": (i32, [vp, C.c_char_p, Dims, C.c_char_p, i32]),
        "msc3d_ctx_gradient": (i32, [vp]),
        "msc3d_ctx_load_codes": (i32, [vp, Dims, vp]),
        "msc3d_ctx_critical": (i32, [vp]),
        "msc3d_ctx_forest": (i32, [vp, i32]),
        "msc3d_ctx_roots": (i32, [vp, i32]),
        "msc3d_ctx_load_parent": (i32, [vp, i32, vp, u64]),
        "msc3d_ctx_se_arcs": (i32, [vp]),
        "msc3d_ctx_load_labels": (i32, [vp, vp, vp]),
        "msc3d_ctx_mark": (i32, [vp, vp, u64]),
        "msc3d_ctx_minor": (i32, [vp]),
        "msc3d_ctx_count": (i32, [vp]),
        "msc3d_ctx_count_minor": (i32, [vp, vp, u64, vp, u64, vp, u64, vp, vp, vp, vp, i32]),
        "msc3d_ctx_compute": (i32, [vp, i32, C.POINTER(C.c_double)]),
        "msc3d_ctx_compute_host": (i32, [vp, i32, C.POINTER(C.c_double), C.POINTER(HostOutputs)]),
        "msc3d_ctx_deliver_host": (i32, [vp, C.POINTER(HostOutputs)]),
        "msc3d_ctx_bind_codes": (i32, [vp, Dims, vp]),
        "msc3d_ctx_compute_host_values": (i32, [vp, Dims, i32, vp, i32, C.POINTER(C.c_double), C.POINTER(HostOutputs)]),
        "msc3d_ctx_compute_codes": (i32, [vp, i32, C.c_uint32, C.c_uint32, C.POINTER(C.c_double)]),
        "msc3d_ctx_cp_values": (i32, [vp]),
        "msc3d_ctx_validate_gradient": (i32, [vp, u64, C.POINTER(u64)]),
        "msc3d_ctx_boundary_check": (i32, [vp, C.POINTER(u64)]),
        "msc3d_boundary_check_host": (i32, [vp, u64, vp, u64, vp, vp, vp, C.POINTER(u64)]),
        "msc3d_mg_plan": (i32, [i64, i32, i32, C.POINTER(i64)]),
        "msc3d_nccl_unique_id": (i32, [C.POINTER(C.c_uint8)]),
        "msc3d_comm_create_nccl": (i32, [C.POINTER(vp), C.POINTER(C.c_uint8), i32, i32, i32]),
        "msc3d_comm_create_host": (i32, [C.POINTER(vp), C.POINTER(HostTransport), i32, i32]),
        "msc3d_comm_destroy": (None, [vp]),
        "msc3d_mg_create": (i32, [C.POINTER(vp), vp, i32]),
        "msc3d_mg_destroy": (None, [vp]),
        "msc3d_mg_full_ctx": (vp, [vp]),
        "msc3d_mg_slab_ctx": (vp, [vp]),
        "msc3d_mg_set_stream": (i32, [vp, vp]),
        "msc3d_mg_compute": (i32, [vp, Dims, i32, vp, i32, C.POINTER(C.c_double)]),
        "msc3d_field_hash_f64": (u64, [vp, u64]),
        "msc3d_field_hash_f32": (u64, [vp, u64]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def _raise(status: int, what: str = ""):
    if status == OK:
        return
    msg = lib().msc3d_status_string(status).decode()
    if what:
        msg = f"{what}: {msg}"
    if status == ERR_INVALID:
        raise ValueError(msg)
    if status == ERR_OVERFLOW:
        raise OverflowError(msg)
    if status == ERR_RUNTIME:
        raise RuntimeError(msg)
    if status == ERR_IO:
        raise IoError(msg)
    raise RuntimeError(f"msc3d CUDA failure ({status}): {msg}")


def _dims(d) -> Dims:
    return Dims(int(d[0]), int(d[1]), int(d[2]))


def check_dims(dims, allow_wide=False):
    """GridDims validation (grid.cpp:11-21): ValueError on < 2 per axis or > 2^32-1 cells."""
    _raise(lib().msc3d_check_dims(_dims(dims), int(allow_wide)), "GridDims")


def id_dtype(dims):
    return np.uint32 if lib().msc3d_id_width(_dims(dims)) == 4 else np.uint64


def total_cells(dims):
    return (2 * dims[0] - 1) * (2 * dims[1] - 1) * (2 * dims[2] - 1)


_DT = {1: np.uint8, 2: np.uint16, 4: np.uint32, 8: np.uint64}


class Context:
    """One device context: stream + named device arrays (include/msc3d_cuda.h)."""

    def __init__(self, device: int = 0):
        self._L = lib()
        h = C.c_void_p()
        _raise(self._L.msc3d_ctx_create(C.byref(h), int(device)), "msc3d_ctx_create")
        self.h = h
        self.dims = None
        self.wide = False

    @classmethod
    def borrow(cls, handle, dims=None):
        """A non-owning view of a context created elsewhere (e.g. msc3d_mg_full_ctx)."""
        c = cls.__new__(cls)
        c._L = lib()
        c.h = C.c_void_p(handle)
        c.dims = tuple(dims) if dims else None
        c.wide = False
        c._borrowed = True
        return c

    def close(self):
        if getattr(self, "h", None):
            if not getattr(self, "_borrowed", False):
                self._L.msc3d_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # ---- raw access -------------------------------------------------------------
    def array_info(self, name):
        p, n, e = C.c_void_p(), C.c_uint64(), C.c_int()
        _raise(self._L.msc3d_ctx_array(self.h, name.encode(), C.byref(p), C.byref(n), C.byref(e)), name)
        return p.value, n.value, e.value

    def get(self, name, dtype=None):
        _, n, e = self.array_info(name)
        dt = dtype or _DT[e]
        out = np.empty(n * e // np.dtype(dt).itemsize, dtype=dt)
        _raise(self._L.msc3d_ctx_download(self.h, name.encode(), out.ctypes.data_as(C.c_void_p),
                                          C.c_uint64(out.nbytes)), name)
        return out

    def scalar(self, name):
        v = C.c_int64()
        _raise(self._L.msc3d_ctx_scalar(self.h, name.encode(), C.byref(v)), name)
        return v.value

    def set_option(self, name, value):
        """msc3d_ctx_set_option: "wide_ids" (64-bit id lists on any grid), "kahn_switch_below",
        "exact_batch_rows", "frontier_cap", "term_rank_words", "release_transients", "kahn_async", "side_stream", "d2h_narrow",
        "d2h_escape_cap", "d2h_narrow_max"."""
        _raise(self._L.msc3d_ctx_set_option(self.h, name.encode(), C.c_int64(int(value))), name)
        if name == "wide_ids":
            self.wide = bool(value)
        return self

    def ids(self, dims):
        """dtype of host cell-id arrays this context takes / returns for `dims`."""
        return np.uint64 if self.wide else id_dtype(dims)

    def validate_gradient(self, max_cells_for_cycles=100000):
        """validate_gradient (gradient.hpp:95) of the loaded codes, on the device:
        GradientReport fields as a dict, samples = up to 32 offending cells."""
        out = (C.c_uint64 * 4)()
        _raise(self._L.msc3d_ctx_validate_gradient(self.h, C.c_uint64(max_cells_for_cycles), out),
               "validate_gradient")
        samples = np.sort(self.get("audit_samples", np.uint64))[:32]
        return {"matching_violations": int(out[0]), "cells_in_closed_vpath": int(out[1]),
                "acyclicity_checked": bool(out[2]), "degenerate": bool(out[3]), "samples": samples}

    def boundary_check(self, cp_index=None, arc_src=None, arc_dst=None, arc_mult=None):
        """boundary_check (msc.hpp:101) on the device: odd (top, low) cp-id pairs of the
        last compute's complex, or of the complex given as host arrays."""
        n = C.c_uint64()
        if cp_index is None:
            _raise(self._L.msc3d_ctx_boundary_check(self.h, C.byref(n)), "boundary_check")
        else:
            ci = np.ascontiguousarray(cp_index, dtype=np.uint8)
            a = np.ascontiguousarray(arc_src, dtype=np.uint32)
            b = np.ascontiguousarray(arc_dst, dtype=np.uint32)
            c = np.ascontiguousarray(arc_mult, dtype=np.uint64)
            p = lambda x: x.ctypes.data_as(C.c_void_p)
            _raise(self._L.msc3d_boundary_check_host(self.h, C.c_uint64(ci.size), p(ci), C.c_uint64(a.size), p(a),
                                                     p(b), p(c), C.byref(n)), "boundary_check")
        if n.value == 0:
            return np.zeros((0, 2), np.uint32)
        return np.stack([self.get("odd_top"), self.get("odd_low")], axis=1)

    def cp_values(self):
        """CriticalPoint::value (msc.cpp:106) of the last compute, f64 per critical point."""
        _raise(self._L.msc3d_ctx_cp_values(self.h), "cp_values")
        return self.get("cp_value", np.float64)

    def launches(self):
        return int(self._L.msc3d_ctx_launches(self.h))

    def sync(self):
        _raise(self._L.msc3d_ctx_sync(self.h))

    # ---- stages -----------------------------------------------------------------
    def load_values(self, values, dims):
        v = np.asarray(values)
        vt = VALUE_F64 if v.dtype == np.float64 else VALUE_F32
        v = np.ascontiguousarray(v, dtype=np.float64 if vt == VALUE_F64 else np.float32).ravel()
        if v.size != dims[0] * dims[1] * dims[2]:
            raise ValueError(f"scalar field size {v.size} does not match vertex count")
        self.dims = tuple(int(x) for x in dims)
        _raise(self._L.msc3d_ctx_load_values(self.h, _dims(dims), vt, v.ctypes.data_as(C.c_void_p)),
               "ScalarField")
        return self

    def bind_values(self, device_ptr, dims, value_type=VALUE_F32):
        self.dims = tuple(int(x) for x in dims)
        _raise(self._L.msc3d_ctx_bind_values(self.h, _dims(dims), value_type, C.c_void_p(device_ptr)))
        return self

    def read_volume(self, path, dims, dtype="f64", big_endian=False):
        self.dims = tuple(int(x) for x in dims)
        _raise(self._L.msc3d_ctx_read_volume(self.h, path.encode(), _dims(dims), dtype.encode(),
                                             int(big_endian)), "read_volume")
        return self

    def load_codes(self, codes, dims):
        c = np.ascontiguousarray(codes, dtype=np.uint8)
        if c.size != total_cells(dims):
            raise ValueError("gradient code array size mismatch")
        self.dims = tuple(int(x) for x in dims)
        _raise(self._L.msc3d_ctx_load_codes(self.h, _dims(dims), c.ctypes.data_as(C.c_void_p)))
        return self

    def gradient(self):
        _raise(self._L.msc3d_ctx_gradient(self.h), "assign_gradient")
        return self

    def critical(self):
        _raise(self._L.msc3d_ctx_critical(self.h), "extract_critical_cells")
        return self

    def forest(self, dim):
        _raise(self._L.msc3d_ctx_forest(self.h, int(dim)), "build_forest")
        return self

    def roots(self, dim):
        _raise(self._L.msc3d_ctx_roots(self.h, int(dim)), "find_roots")
        return self

    def load_parent(self, dim, parent):
        p = np.ascontiguousarray(parent, dtype=np.uint32)
        _raise(self._L.msc3d_ctx_load_parent(self.h, int(dim), p.ctypes.data_as(C.c_void_p), C.c_uint64(p.size)))
        return self

    def load_labels(self, l0, l3):
        a = np.ascontiguousarray(l0, dtype=np.uint32)
        b = np.ascontiguousarray(l3, dtype=np.uint32)
        _raise(self._L.msc3d_ctx_load_labels(self.h, a.ctypes.data_as(C.c_void_p), b.ctypes.data_as(C.c_void_p)))
        return self

    def se_arcs(self):
        _raise(self._L.msc3d_ctx_se_arcs(self.h), "saddle_extremum_arcs")
        return self

    def mark(self, sources=None):
        if sources is None:
            _raise(self._L.msc3d_ctx_mark(self.h, None, C.c_uint64(0)), "mark_reachable")
        else:
            s = np.ascontiguousarray(sources, dtype=self.ids(self.dims))
            _raise(self._L.msc3d_ctx_mark(self.h, s.ctypes.data_as(C.c_void_p) if s.size else C.c_void_p(1),
                                          C.c_uint64(s.size)), "mark_reachable")
        return self

    def minor(self):
        _raise(self._L.msc3d_ctx_minor(self.h), "build_minor")
        return self

    def count(self):
        _raise(self._L.msc3d_ctx_count(self.h), "count_paths")
        return self

    def compute(self, options=OPT_SEGMENTATION):
        ms = (C.c_double * 5)()
        _raise(self._L.msc3d_ctx_compute(self.h, int(options), ms), "compute")
        return list(ms)


# ---------------------------------------------------------------------------------
# Reference-shaped API (proj/include/msc3d/*.hpp); every call runs on the GPU.
# ---------------------------------------------------------------------------------

@dataclass
class GradientField:
    """gradient.hpp:43-63: dims + one pair-code byte per cell."""
    dims: tuple
    code: np.ndarray


@dataclass
class CriticalCells:
    """gradient.hpp:69-78: four ascending id lists."""
    by_dim: list

    def euler(self):
        return len(self.by_dim[0]) - len(self.by_dim[1]) + len(self.by_dim[2]) - len(self.by_dim[3])


@dataclass
class RootLabels:
    label: np.ndarray
    rounds: int


@dataclass
class MSComplex:
    """msc.hpp:53-66 as flat arrays (cp ids are positions)."""
    dims: tuple
    cp_cell: np.ndarray
    cp_index: np.ndarray
    arc_src: np.ndarray
    arc_dst: np.ndarray
    arc_mult: np.ndarray
    input_hash: int = 0
    labels_min: Optional[np.ndarray] = None
    labels_max: Optional[np.ndarray] = None
    stage_ms: list = field(default_factory=list)

    def euler(self):
        return int(np.sum(np.where(self.cp_index % 2 == 1, -1, 1)))

    def count_by_index(self, i):
        return int(np.sum(self.cp_index == i))


def _ctx(ctx):
    return ctx if ctx is not None else Context()


def assign_gradient(values, dims, ctx=None) -> GradientField:
    """assign_gradient (gradient.hpp:66)."""
    c = _ctx(ctx)
    c.load_values(values, dims).gradient()
    return GradientField(tuple(dims), c.get("codes"))


def extract_critical_cells(g: GradientField, ctx=None) -> CriticalCells:
    """extract_critical_cells (gradient.hpp:80)."""
    c = _ctx(ctx)
    c.load_codes(g.code, g.dims).critical()
    return CriticalCells([c.get(f"crit{k}") for k in range(4)])


def build_forest(g: GradientField, dim: int, ctx=None) -> np.ndarray:
    """build_forest (extrema.hpp:48): parent per vertex (dim 0) or cube (dim 3)."""
    if dim not in (0, 3):
        raise ValueError("build_forest: dim must be 0 or 3")
    c = _ctx(ctx)
    c.load_codes(g.code, g.dims).forest(dim)
    return c.get("parent0" if dim == 0 else "parent3")


def find_roots(parent, ctx=None, dims=(2, 2, 2)) -> RootLabels:
    """find_roots (extrema.hpp:56): synchronous pointer doubling, exact round count."""
    c = _ctx(ctx)
    if c.dims is None:
        c.load_codes(np.ones(total_cells(dims), np.uint8), dims)
    c.load_parent(0, parent).roots(0)
    return RootLabels(c.get("label0"), c.scalar("rounds0"))


def saddle_extremum_arcs(g: GradientField, labels0, labels3, ctx=None):
    """saddle_extremum_arcs (extrema.hpp:67): (saddle, extremum, multiplicity) arrays."""
    c = _ctx(ctx)
    c.load_codes(g.code, g.dims).load_labels(labels0, labels3).se_arcs()
    return c.get("se_saddle"), c.get("se_extremum"), c.get("se_mult")


def mark_reachable(g: GradientField, one_saddles=None, ctx=None):
    """mark_reachable (saddle_graph.hpp:51): marked bytes, one_saddles, two_saddles."""
    c = _ctx(ctx)
    c.load_codes(g.code, g.dims).mark(one_saddles)
    return c.get("marked"), c.get("one_saddles"), c.get("two_saddles")


def compute(values, dims, with_segmentation=True, ctx=None, hash_input=True) -> MSComplex:
    """compute (msc.hpp:87): the whole pipeline on the GPU."""
    c = _ctx(ctx)
    v = np.asarray(values)
    c.load_values(v, dims)
    ms = c.compute(OPT_SEGMENTATION if with_segmentation else 0)
    h = 0
    if hash_input:
        L = lib()
        if v.dtype == np.float64:
            vv = np.ascontiguousarray(v, dtype=np.float64).ravel()
            h = int(L.msc3d_field_hash_f64(vv.ctypes.data_as(C.c_void_p), C.c_uint64(vv.size)))
        else:
            vv = np.ascontiguousarray(v, dtype=np.float32).ravel()
            h = int(L.msc3d_field_hash_f32(vv.ctypes.data_as(C.c_void_p), C.c_uint64(vv.size)))
    m = MSComplex(tuple(dims), c.get("cp_cell"), c.get("cp_index"), c.get("arc_src"),
                  c.get("arc_dst"), c.get("arc_mult"), h, stage_ms=ms)
    if with_segmentation:
        m.labels_min = c.get("labels_min")
        m.labels_max = c.get("labels_max")
    return m


def synth(kind: str, dims, seed: int = 1, threads: int = 0) -> np.ndarray:
    """Canonical synthetic f32 field: gauss | gnoise | noise."""
    L = C.CDLL(SYNTH_PATH)
    out = np.empty(int(dims[0]) * int(dims[1]) * int(dims[2]), dtype=np.float32)
    rc = L.msc3d_synth_f32(kind.encode(), C.c_int64(dims[0]), C.c_int64(dims[1]), C.c_int64(dims[2]),
                           C.c_uint64(seed), out.ctypes.data_as(C.c_void_p), C.c_int(threads))
    if rc != 0:
        raise ValueError(f"unknown field kind {kind!r}")
    return out

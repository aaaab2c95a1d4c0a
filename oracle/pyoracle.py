"""Test infrastructure: ctypes access to the two CPU checkers.

* ``Ref``      -- the UNMODIFIED reference library (``oracle/_ref/libmsc3d_ref_capi.so``,
                  built from /root/reference/proj/src by ``oracle/Makefile``).
* ``Oracle64`` -- our serial restatement with 64-bit cell ids (``oracle/_lib/liboracle64.so``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s reference /
cpu_baseline arm may import this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libmsc3d_ref_capi.so")
ORC_SO = os.path.join(HERE, "_lib", "liboracle64.so")

STATUS_NAMES = {0: "ok", 1: "invalid_argument", 2: "overflow_error", 3: "runtime_error",
                4: "exception", 5: "io_error"}


class CheckerError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status
        self.kind = STATUS_NAMES.get(status, str(status))


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


class _Bundle:
    def __init__(self, lib, prefix, handle):
        self._lib, self._p, self._h = lib, prefix, handle

    def __del__(self):
        try:
            getattr(self._lib, self._p + "_bundle_free")(self._h)
        except Exception:
            pass

    def status(self):
        return getattr(self._lib, self._p + "_bundle_status")(self._h)

    def error(self):
        return getattr(self._lib, self._p + "_bundle_error")(self._h).decode()

    def check(self):
        s = self.status()
        if s != 0:
            raise CheckerError(s, self.error())
        return self

    def has(self, name):
        d = C.c_void_p()
        n = C.c_uint64()
        return getattr(self._lib, self._p + "_bundle_get")(self._h, name.encode(), C.byref(d), C.byref(n)) == 0

    def get(self, name, dtype):
        d = C.c_void_p()
        n = C.c_uint64()
        rc = getattr(self._lib, self._p + "_bundle_get")(self._h, name.encode(), C.byref(d), C.byref(n))
        if rc != 0:
            raise KeyError(name)
        nbytes = n.value
        if nbytes == 0:
            return np.zeros(0, dtype=dtype)
        buf = (C.c_uint8 * nbytes).from_address(d.value)
        return np.frombuffer(bytes(buf), dtype=dtype).copy()


class _Checker:
    SO = None
    PREFIX = None

    def __init__(self):
        if not os.path.exists(self.SO):
            raise FileNotFoundError(f"{self.SO} missing: run `make -C oracle`")
        self.lib = C.CDLL(self.SO)
        for name in ("bundle_get", "bundle_status", "bundle_free", "bundle_names"):
            getattr(self.lib, f"{self.PREFIX}_{name}")
        getattr(self.lib, f"{self.PREFIX}_bundle_error").restype = C.c_char_p
        for fn in self._FUNCS:
            f = getattr(self.lib, f"{self.PREFIX}_{fn}")
            f.restype = C.c_void_p
        self.lib.__getattr__  # noqa

    def _call(self, fn, *args):
        f = getattr(self.lib, f"{self.PREFIX}_{fn}")
        h = f(*args)
        return _Bundle(self.lib, self.PREFIX, h).check()

    # ---- shared API (same argument conventions in both checkers) -------------------
    def gradient(self, values, dims, threads=0):
        v = np.ascontiguousarray(values, dtype=np.float64)
        b = self._call("gradient", _ptr(v), C.c_int64(dims[0]), C.c_int64(dims[1]),
                       C.c_int64(dims[2]), C.c_int(threads))
        return b.get("codes", np.uint8)

    def critical(self, codes, dims, threads=0):
        c = np.ascontiguousarray(codes, dtype=np.uint8)
        b = self._call("critical", _ptr(c), C.c_int64(dims[0]), C.c_int64(dims[1]),
                       C.c_int64(dims[2]), C.c_int(threads))
        return [b.get(f"c{k}", self.ID) for k in range(4)]

    def forest(self, codes, dims, dim, threads=0):
        c = np.ascontiguousarray(codes, dtype=np.uint8)
        b = self._call("forest", _ptr(c), C.c_int64(dims[0]), C.c_int64(dims[1]),
                       C.c_int64(dims[2]), C.c_int(dim), C.c_int(threads))
        return b.get("parent", self.ID)

    def roots(self, parent, threads=0):
        p = np.ascontiguousarray(parent, dtype=self.ID)
        b = self._call("roots", _ptr(p), C.c_uint64(len(p)), C.c_int(threads))
        return b.get("label", self.ID), int(b.get("rounds", np.int32)[0])

    def se_arcs(self, codes, dims, l0, l3, threads=0):
        c = np.ascontiguousarray(codes, dtype=np.uint8)
        a0 = np.ascontiguousarray(l0, dtype=self.ID)
        a3 = np.ascontiguousarray(l3, dtype=self.ID)
        b = self._call("se_arcs", _ptr(c), C.c_int64(dims[0]), C.c_int64(dims[1]),
                       C.c_int64(dims[2]), _ptr(a0), _ptr(a3), C.c_int(threads))
        return b.get("saddle", self.ID), b.get("extremum", self.ID), b.get("mult", np.uint32)

    def mark(self, codes, dims, sources, threads=0):
        c = np.ascontiguousarray(codes, dtype=np.uint8)
        s = np.ascontiguousarray(sources, dtype=self.ID)
        b = self._call("mark", _ptr(c), C.c_int64(dims[0]), C.c_int64(dims[1]),
                       C.c_int64(dims[2]), _ptr(s), C.c_uint64(len(s)), C.c_int(threads))
        return b.get("marked", np.uint8), b.get("one_saddles", self.ID), b.get("two_saddles", self.ID)

    def minor(self, codes, dims, marked, ones, twos, threads=0):
        c = np.ascontiguousarray(codes, dtype=np.uint8)
        m = np.ascontiguousarray(marked, dtype=np.uint8)
        o = np.ascontiguousarray(ones, dtype=self.ID)
        t = np.ascontiguousarray(twos, dtype=self.ID)
        b = self._call("minor", _ptr(c), C.c_int64(dims[0]), C.c_int64(dims[1]),
                       C.c_int64(dims[2]), _ptr(m), _ptr(o), C.c_uint64(len(o)), _ptr(t),
                       C.c_uint64(len(t)), C.c_int(threads))
        out = {k: b.get(k, self.ID) for k in ("one_saddles", "junctions", "two_saddles")}
        for k in ("s1_to_j", "j_to_j", "j_to_s2", "s1_to_s2"):
            out[k] = (b.get(k + ".src", np.uint32), b.get(k + ".dst", np.uint32),
                      b.get(k + ".mult", np.uint64))
        return out

    def count_paths(self, minor, threads=0):
        keep = []

        def arr(x, dt):
            a = np.ascontiguousarray(x, dtype=dt)
            keep.append(a)
            return a

        ones = arr(minor["one_saddles"], self.ID)
        juncs = arr(minor["junctions"], self.ID)
        twos = arr(minor["two_saddles"], self.ID)
        names = ("s1_to_j", "j_to_j", "j_to_s2", "s1_to_s2")
        srcs = (C.c_void_p * 4)(*[_ptr(arr(minor[k][0], np.uint32)) for k in names])
        dsts = (C.c_void_p * 4)(*[_ptr(arr(minor[k][1], np.uint32)) for k in names])
        mults = (C.c_void_p * 4)(*[_ptr(arr(minor[k][2], np.uint64)) for k in names])
        counts = (C.c_uint64 * 4)(*[len(minor[k][0]) for k in names])
        b = self._call("count_paths", _ptr(ones), C.c_uint64(len(ones)), _ptr(juncs),
                       C.c_uint64(len(juncs)), _ptr(twos), C.c_uint64(len(twos)), srcs, dsts,
                       mults, counts, C.c_int(threads))
        return b.get("one_saddle", self.ID), b.get("two_saddle", self.ID), b.get("paths", np.uint64)

    def compute(self, values, dims, threads=0, with_segmentation=True, validate=False,
                dtype="f32", want_text=False):
        v = np.ascontiguousarray(values, dtype=np.float64)
        b = self._call("compute", _ptr(v), C.c_int64(dims[0]), C.c_int64(dims[1]),
                       C.c_int64(dims[2]), C.c_int(threads), C.c_int(int(with_segmentation)),
                       C.c_int(int(validate)), dtype.encode(), C.c_int(int(want_text)))
        out = {
            "cp_cell": b.get("cp_cell", self.ID),
            "cp_index": b.get("cp_index", np.int32),
            "cp_value": b.get("cp_value", np.float64),
            "arc_src": b.get("arc_src", np.uint32),
            "arc_dst": b.get("arc_dst", np.uint32),
            "arc_mult": b.get("arc_mult", np.uint64),
            "input_hash": int(b.get("input_hash", np.uint64)[0]),
            "timings": b.get("timings", np.float64),
            "wall": float(b.get("wall", np.float64)[0]),
            "hash_seconds": float(b.get("hash_seconds", np.float64)[0]),
        }
        if b.has("labels_min"):
            out["labels_min"] = b.get("labels_min", np.uint32)
            out["labels_max"] = b.get("labels_max", np.uint32)
        for k in ("json", "cp_csv", "arcs_csv", "labels_min_bytes"):
            if b.has(k):
                out[k] = b.get(k, np.uint8).tobytes()
        if b.has("boundary_odd_pairs"):
            out["boundary_odd_pairs"] = int(b.get("boundary_odd_pairs", np.uint64)[0])
        return out


class Ref(_Checker):
    """The compiled, unmodified reference (32-bit cell ids)."""
    SO = REF_SO
    PREFIX = "ref"
    ID = np.uint32
    _FUNCS = ("gradient", "validate_gradient", "critical", "forest", "roots", "se_arcs",
              "successors", "mark", "minor", "count_paths", "read_volume", "generate", "compute")

    def __init__(self):
        super().__init__()
        self.lib.ref_field_hash.restype = C.c_uint64
        self.lib.ref_max_vertex_of.restype = C.c_uint32

    def generate(self, kind, dims, seed):
        b = self._call("generate", kind.encode(), C.c_int64(dims[0]), C.c_int64(dims[1]),
                       C.c_int64(dims[2]), C.c_uint64(seed))
        return b.get("values", np.float64)

    def field_hash(self, values):
        v = np.ascontiguousarray(values, dtype=np.float64)
        return int(self.lib.ref_field_hash(_ptr(v), C.c_uint64(len(v))))

    def validate_gradient(self, codes, dims, max_cells=100000):
        c = np.ascontiguousarray(codes, dtype=np.uint8)
        b = self._call("validate_gradient", _ptr(c), C.c_int64(dims[0]), C.c_int64(dims[1]),
                       C.c_int64(dims[2]), C.c_uint64(max_cells))
        return {k: int(b.get(k, np.uint64 if "_" in k and k != "acyclicity_checked" else np.uint8)[0])
                for k in ("matching_violations", "cells_in_closed_vpath")}

    def successors(self, codes, dims, edge):
        c = np.ascontiguousarray(codes, dtype=np.uint8)
        b = self._call("successors", _ptr(c), C.c_int64(dims[0]), C.c_int64(dims[1]),
                       C.c_int64(dims[2]), C.c_uint32(edge))
        return list(zip(b.get("kind", np.uint8).tolist(), b.get("cell", np.uint32).tolist()))

    def read_volume(self, path, dims, dtype, big_endian=False):
        b = self._call("read_volume", path.encode(), C.c_int64(dims[0]), C.c_int64(dims[1]),
                       C.c_int64(dims[2]), dtype.encode(), C.c_int(int(big_endian)))
        return b.get("values", np.float64)


class Oracle64(_Checker):
    """Our serial restatement (64-bit cell ids), oracle/oracle64.cpp."""
    SO = ORC_SO
    PREFIX = "orc"
    ID = np.uint64
    _FUNCS = ("gradient", "critical", "forest", "roots", "se_arcs", "mark", "minor",
              "count_paths", "compute")


def synth_lib():
    """The product's input synthesizer (not a checker; re-exported for convenience)."""
    root = os.path.dirname(HERE)
    return os.path.join(root, "paper_2009_03707_b200", "lib", "libmsc3d_synth.so")

"""Multi-GPU MS complex: the Python side of the C++ orchestrator (csrc/multigpu.cu).

One process per GPU.  The step itself -- P2P halo exchange, z-slab gradient, per-slab
critical compaction with count/list gathers, allgather-v of the owned code planes,
extrema on the replicated codes, reachability + counting from the rank's 1-saddle
slice, allgather-v of the arc blocks -- runs in C++ (msc3d_mg_compute) over a
communicator:

* NCCL (``transport="nccl"``, production: torchrun, one GPU per rank): rank 0 draws the
  ncclUniqueId through the C ABI, torch.distributed broadcasts it, every rank builds its
  communicator in C++ (libnccl.so.2, the library torch.distributed also loads);
* host (``transport="host"``): the orchestrator's collectives are allgathers over host
  buffers, implemented here with torch.distributed (gloo) -- several ranks on one GPU in
  the tests.

No step changes any result: every rank ends with the same complex as a single-GPU
compute() (tests/test_multigpu.py).  SURVEY.md §8(e), DESIGN.md §5.
"""
from __future__ import annotations

import ctypes as C
import sys
import traceback
from dataclasses import dataclass

import numpy as np

HALO = 2  # vertex planes of halo on each side of a slab (multigpu.cu kHalo)


@dataclass(frozen=True)
class SlabPlan:
    rank: int
    world: int
    nz: int
    z0: int          # owned vertex planes [z0, z1)
    z1: int
    lo: int          # slab grid (with halo): vertex planes [lo, hi)
    hi: int
    own_c0: int      # owned global lattice planes [own_c0, own_c1)
    own_c1: int
    local_c0: int    # first owned lattice plane in the slab grid's lattice

    @property
    def local_nz(self) -> int:
        return self.hi - self.lo


def slab_plan(nz: int, world: int, rank: int) -> SlabPlan:
    """msc3d_mg_plan: vertex planes split as evenly as possible (>= 2 per rank)."""
    from . import _raise, lib
    out = (C.c_int64 * 7)()
    _raise(lib().msc3d_mg_plan(int(nz), int(world), int(rank), out), "msc3d_mg_plan")
    return SlabPlan(rank, world, nz, *[int(x) for x in out])


def source_slice(c1: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced slice [first, first + count) of the critical 1-cells
    (stages.cu: compute_from_codes, sharded)."""
    first = c1 * rank // world
    return first, c1 * (rank + 1) // world - first


def slab_values(values: np.ndarray, dims, plan: SlabPlan, own_only: bool = True) -> np.ndarray:
    """This rank's samples out of the whole field: its own vertex planes [z0, z1)
    (what msc3d_mg_compute takes), or the whole slab grid [lo, hi)."""
    nx, ny, nz = dims
    v = np.asarray(values).reshape(nz, ny, nx)
    a, b = (plan.z0, plan.z1) if own_only else (plan.lo, plan.hi)
    return np.ascontiguousarray(v[a:b]).reshape(-1)


class HostTransport:
    """msc3d_host_transport over torch.distributed (any backend with CPU tensors: gloo):
    the orchestrator's only host primitive, an allgather of equal-size byte blocks."""

    def __init__(self, group=None):
        from . import ALLGATHER_FN, HostTransport as _HT
        self.group = group
        self.calls = 0
        self._fn = ALLGATHER_FN(self._allgather)  # kept alive as long as the transport
        self.struct = _HT(None, self._fn)

    def allgather_bytes(self, data: bytes) -> bytes:
        import torch
        import torch.distributed as dist
        world = dist.get_world_size(self.group)
        n = len(data)
        if n == 0:
            return b""
        t = torch.frombuffer(bytearray(data), dtype=torch.uint8)
        out = [torch.empty(n, dtype=torch.uint8) for _ in range(world)]
        dist.all_gather(out, t, group=self.group)
        return b"".join(o.numpy().tobytes() for o in out)

    def _allgather(self, user, send, recv, nbytes):
        try:
            self.calls += 1
            data = C.string_at(send, nbytes) if nbytes else b""
            got = self.allgather_bytes(data)
            if got:
                C.memmove(recv, got, len(got))
            return 0
        except Exception:  # pragma: no cover - reported to the C side as a failure
            traceback.print_exc(file=sys.stderr)
            return 1


class MultiGPU:
    """One rank of a multi-GPU compute: communicator + the orchestrator's two contexts
    (slab grid, whole grid).  step(own) runs msc3d_mg_compute on this rank's own vertex
    planes (a device pointer or a CUDA torch tensor)."""

    def __init__(self, dims, rank: int, world: int, device: int = 0, transport: str = "nccl", group=None):
        from . import Context, _raise, lib
        self._L = lib()
        self.dims = tuple(int(x) for x in dims)
        self.rank, self.world = rank, world
        self.plan = slab_plan(self.dims[2], world, rank)
        self.transport = None
        comm = C.c_void_p()
        if transport == "nccl":
            import torch.distributed as dist
            uid = (C.c_uint8 * 128)()
            if rank == 0:
                _raise(self._L.msc3d_nccl_unique_id(uid), "ncclGetUniqueId")
            box = [bytes(uid)]
            if world > 1:
                dist.broadcast_object_list(box, src=0, group=group)
            uid = (C.c_uint8 * 128).from_buffer_copy(box[0])
            _raise(self._L.msc3d_comm_create_nccl(C.byref(comm), uid, rank, world, device), "ncclCommInitRank")
        elif transport == "host":
            self.transport = HostTransport(group)
            _raise(self._L.msc3d_comm_create_host(C.byref(comm), C.byref(self.transport.struct), rank, world),
                   "msc3d_comm_create_host")
        else:
            raise ValueError(f"unknown transport {transport!r}")
        self.comm = comm
        mg = C.c_void_p()
        _raise(self._L.msc3d_mg_create(C.byref(mg), comm, int(device)), "msc3d_mg_create")
        self.mg = mg
        self.full = Context.borrow(self._L.msc3d_mg_full_ctx(mg), self.dims)
        self.slab = Context.borrow(self._L.msc3d_mg_slab_ctx(mg))
        self.stage_ms = [0.0] * 7

    def set_stream(self, stream_ptr: int):
        from . import _raise
        _raise(self._L.msc3d_mg_set_stream(self.mg, C.c_void_p(stream_ptr)), "set_stream")

    def step(self, own_values, options: int = 1, value_type: int | None = None):
        from . import VALUE_F32, VALUE_F64, _dims, _raise
        ptr = own_values.data_ptr() if hasattr(own_values, "data_ptr") else int(own_values)
        if value_type is None:
            value_type = VALUE_F64 if str(getattr(own_values, "dtype", "")).endswith("float64") else VALUE_F32
        st = (C.c_double * 7)()
        _raise(self._L.msc3d_mg_compute(self.mg, _dims(self.dims), int(value_type), C.c_void_p(ptr), int(options), st),
               "msc3d_mg_compute")
        self.stage_ms = list(st)
        return self.stage_ms

    def outputs(self, names=("cp_cell", "cp_index", "arc_src", "arc_dst", "arc_mult", "labels_min", "labels_max")):
        """The assembled complex (host copies)."""
        out = {}
        for k in names:
            try:
                out[k] = self.full.get(k)
            except Exception:
                if k.startswith("labels"):
                    continue
                raise
        return out

    def device_arrays(self, names=("cp_cell", "cp_index", "arc_src", "arc_dst", "arc_mult", "labels_min",
                                   "labels_max")):
        """Zero-copy torch views of the assembled complex on this rank's GPU."""
        out = {}
        for k in names:
            ptr, n, e = self.full.array_info(k)
            out[k] = _wrap_device(ptr, n * e) if n else None
        return out

    def launches(self) -> int:
        return self.full.launches()

    def close(self):
        if getattr(self, "mg", None):
            self.full.close()
            self.slab.close()
            self._L.msc3d_mg_destroy(self.mg)
            self.mg = None
        if getattr(self, "comm", None):
            self._L.msc3d_comm_destroy(self.comm)
            self.comm = None


def _wrap_device(ptr: int, nbytes: int):
    """A torch uint8 view of device memory owned by a context (no copy)."""
    import torch

    class _Arr:
        __cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3}

    return torch.as_tensor(_Arr(), device="cuda")

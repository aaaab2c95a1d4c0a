"""Multi-GPU MS complex: z-slab gradient with halos, replicated codes, 1-saddle-sharded
saddle stages, allgather-v of the arcs (BASELINE.json north_star).

One process per GPU (torch.distributed, NCCL over NVLink; gloo on CPU for the host
logic tests).  Per step, rank r of G:

1. gradient on its z-slab of vertex planes [z0, z1) plus a 2-plane halo on each side
   (values of planes [z0-2, z1+2) ∩ [0, nz)).  A vertex's lower star lies in its
   3x3x3 neighbourhood (gradient.cpp:13-20), so every vertex of [z0-1, z1+1) gets its
   exact star, hence every cell of lattice planes [2 z0 - 1, 2 z1] its exact code --
   in particular all of the rank's own lattice planes [2 z0, 2 z1) (last rank: up to
   ez).  Vertex ids are shifted on the slab, which the tie-break tolerates (it only
   compares ids, and the shift preserves their order).
2. allgather of the owned code planes (N/G bytes per rank): every rank holds the
   whole GradientField (the north star's "replicated gradient field").
3. critical cells and extrema on the replicated codes (cheap, replicated).
4. reachability + path counting from a contiguous slice of the critical 1-cells
   (crit1 is sorted by cell id, so an index slice is a z-slab of sources): the 1s->2s
   arcs of those 1-saddles are a contiguous block of the global sorted arc list.
5. allgather-v of the arc blocks; the complex is assembled identically on every rank.

No step changes any result: the assembled complex equals the single-GPU compute()
(tests/test_multigpu.py checks it on one GPU by running the shards in sequence, and the
collectives' host logic on CPU with gloo, world_size 2).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

HALO = 2  # vertex planes of halo on each side of a slab


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


def slab_plan(nz: int, world: int, rank: int, halo: int = HALO) -> SlabPlan:
    """Vertex planes split as evenly as possible; every rank gets >= 1 plane."""
    if nz < 2:
        raise ValueError("nz must be >= 2 (grid.cpp:13-16)")
    if world > nz:
        raise ValueError("more ranks than vertex planes")
    z0 = nz * rank // world
    z1 = nz * (rank + 1) // world
    lo = max(0, z0 - halo)
    hi = min(nz, z1 + halo)
    ez = 2 * nz - 1
    own_c0 = 2 * z0
    own_c1 = ez if rank == world - 1 else 2 * z1
    return SlabPlan(rank, world, nz, z0, z1, lo, hi, own_c0, own_c1, own_c0 - 2 * lo)


def source_slice(c1: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced slice [first, first + count) of the critical 1-cells."""
    first = c1 * rank // world
    return first, c1 * (rank + 1) // world - first


# ---------------------------------------------------------------------------------
# collectives (torch.distributed; the same code runs on NCCL and on gloo)
# ---------------------------------------------------------------------------------
def allgather_equal(chunk, group=None):
    """Concatenate equal-size 1-D chunks of every rank in rank order."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    if chunk.device.type == "cuda" and dist.get_backend(group) != "nccl":
        # gloo (tests: several ranks sharing one GPU) gathers through host memory
        return allgather_equal(chunk.cpu(), group).to(chunk.device)
    out = torch.empty(world * chunk.numel(), dtype=chunk.dtype, device=chunk.device)
    if chunk.device.type == "cuda":
        dist.all_gather_into_tensor(out, chunk.contiguous(), group=group)
    else:
        dist.all_gather(list(out.chunk(world)), chunk.contiguous(), group=group)
    return out


def allgather_v(t, group=None):
    """allgather-v of a 1-D tensor (NCCL has no native allgather-v): sizes first,
    then one equal-size allgather of the padded blocks, then the padding is dropped."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    n = torch.tensor([t.numel()], dtype=torch.int64, device=t.device)
    sizes = allgather_equal(n, group).tolist()
    m = max(sizes)
    pad = torch.zeros(m, dtype=t.dtype, device=t.device)
    pad[: t.numel()] = t
    g = allgather_equal(pad, group).view(world, m)
    return torch.cat([g[r, : sizes[r]] for r in range(world)]) if world > 1 else g[0, : sizes[0]]


def gather_codes(local_codes, plan: SlabPlan, plane_bytes: int, chunk_planes: int, group=None):
    """Owned lattice planes of every rank -> the whole GradientField (1-D uint8).
    local_codes: the slab grid's code array (1-D uint8 tensor)."""
    import torch
    own = plan.own_c1 - plan.own_c0
    a = plan.local_c0 * plane_bytes
    chunk = torch.zeros(chunk_planes * plane_bytes, dtype=torch.uint8, device=local_codes.device)
    chunk[: own * plane_bytes] = local_codes[a: a + own * plane_bytes]
    g = allgather_equal(chunk, group)
    ez = 2 * plan.nz - 1
    world = plan.world
    # every rank but possibly the last owns exactly chunk_planes planes when nz is
    # divisible by the world size: then the gathered buffer is already contiguous
    parts = []
    for r in range(world):
        p = slab_plan(plan.nz, world, r)
        n = (p.own_c1 - p.own_c0) * plane_bytes
        parts.append(g[r * chunk_planes * plane_bytes: r * chunk_planes * plane_bytes + n])
    codes = torch.cat(parts)
    assert codes.numel() == ez * plane_bytes
    return codes


def chunk_planes_for(nz: int, world: int) -> int:
    return max(slab_plan(nz, world, r).own_c1 - slab_plan(nz, world, r).own_c0 for r in range(world))


# ---------------------------------------------------------------------------------
# one sharded step on this rank
# ---------------------------------------------------------------------------------
class ShardedCompute:
    """Holds the two device contexts of a rank (slab grid, whole grid) and runs one
    multi-GPU step.  values_slab: device f32 tensor of the slab grid's vertices
    (planes [plan.lo, plan.hi))."""

    def __init__(self, m, dims, plan: SlabPlan, device: int, group=None):
        self.m = m
        self.dims = tuple(dims)
        self.plan = plan
        self.group = group
        self.slab = m.Context(device)
        self.full = m.Context(device)
        self.ex = 2 * dims[0] - 1
        self.ey = 2 * dims[1] - 1
        self.plane_bytes = self.ex * self.ey
        self.chunk_planes = chunk_planes_for(dims[2], plan.world)

    def set_stream(self, stream_ptr):
        for c in (self.slab, self.full):
            c._L.msc3d_ctx_set_stream(c.h, C.c_void_p(stream_ptr))

    def _device_array(self, ctx, name, dtype):
        import torch
        ptr, n, e = ctx.array_info(name)
        if n == 0:
            return torch.empty(0, dtype=dtype, device="cuda")
        return _wrap_device(ptr, n * e, torch.uint8).view(dtype)

    def step(self, values_slab, options=1):
        """Returns dict of device tensors of the assembled complex (identical on every rank)."""
        import torch
        m, plan = self.m, self.plan
        nx, ny, nz = self.dims
        ldims = (nx, ny, plan.local_nz)
        m._raise(self.slab._L.msc3d_ctx_bind_values(self.slab.h, m.Dims(*ldims), m.VALUE_F32,
                                                     C.c_void_p(values_slab.data_ptr())), "bind_values")
        m._raise(self.slab._L.msc3d_ctx_gradient(self.slab.h), "gradient")
        self.slab.sync()  # the contexts' stream -> torch's (collectives, copies)
        local_codes = self._device_array(self.slab, "codes", torch.uint8)
        codes = gather_codes(local_codes, plan, self.plane_bytes, self.chunk_planes, self.group)
        torch.cuda.current_stream().synchronize()
        m._raise(self.full._L.msc3d_ctx_bind_codes(self.full.h, m.Dims(*self.dims), C.c_void_p(codes.data_ptr())),
                 "bind_codes")
        st = (C.c_double * 5)()
        m._raise(self.full._L.msc3d_ctx_compute_codes(self.full.h, options, plan.rank, plan.world, st),
                 "compute_codes")
        self.full.sync()
        out = {k: self._device_array(self.full, k, torch.uint8) for k in ("cp_cell", "cp_index")}
        if plan.world == 1:
            for k, dt in (("arc_src", torch.int32), ("arc_dst", torch.int32), ("arc_mult", torch.int64)):
                out[k] = self._device_array(self.full, k, dt)
        else:
            for k, dt in (("src", torch.int32), ("dst", torch.int32), ("mult", torch.int64)):
                a = self._device_array(self.full, "arcA_" + k, dt)
                b = allgather_v(self._device_array(self.full, "arcB_" + k, dt), self.group)
                c = self._device_array(self.full, "arcC_" + k, dt)
                out["arc_" + k] = torch.cat([a, b, c])
        if options & m.OPT_SEGMENTATION:
            out["labels_min"] = self._device_array(self.full, "labels_min", torch.int32)
            out["labels_max"] = self._device_array(self.full, "labels_max", torch.int32)
        self.stage_ms = list(st)
        return out

    def close(self):
        self.slab.close()
        self.full.close()


def _wrap_device(ptr: int, nbytes: int, dtype):
    """A torch view of device memory owned by a context (no copy)."""
    import torch

    class _Arr:
        __cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3}

    return torch.as_tensor(_Arr(), device="cuda")


def slab_values(values: np.ndarray, dims, plan: SlabPlan) -> np.ndarray:
    """The slab grid's samples (x-fastest) out of the whole field."""
    nx, ny, nz = dims
    v = np.asarray(values).reshape(nz, ny, nx)
    return np.ascontiguousarray(v[plan.lo: plan.hi]).reshape(-1)

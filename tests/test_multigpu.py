"""Multi-GPU decomposition (csrc/multigpu.cu + paper_2009_03707_b200/multigpu.py,
SURVEY.md §8(e)).

* CPU: the slab plan (msc3d_mg_plan, host-only C ABI), the host transport's allgather
  over gloo with world_size 2 -- called through the C function pointer the orchestrator
  uses.
* GPU (one device): z-slab gradients with 2-plane halos stitched into the whole
  GradientField equal the single-GPU codes byte for byte; the C++ orchestrator
  (msc3d_mg_compute: halo exchange, slab gradient, per-slab critical compaction, code /
  list / arc gathers, 1-saddle-sharded saddle stages) run by 2 and 3 processes sharing
  the GPU over the host transport (gloo), and by one rank over NCCL, reassembles the
  single-GPU complex exactly.
"""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2009_03707_b200 as m
from paper_2009_03707_b200 import multigpu as mg


def test_slab_plan_covers_lattice():
    for nz in (2, 4, 7, 16, 64, 512):
        for world in (1, 2, 3, 4, 8):
            if world > 1 and nz // world < mg.HALO:
                with pytest.raises(ValueError):
                    mg.slab_plan(nz, world, 0)
                continue
            plans = [mg.slab_plan(nz, world, r) for r in range(world)]
            assert plans[0].own_c0 == 0 and plans[-1].own_c1 == 2 * nz - 1
            for a, b in zip(plans, plans[1:]):
                assert a.own_c1 == b.own_c0 and a.z1 == b.z0
            for p in plans:
                assert p.z1 - p.z0 >= (mg.HALO if world > 1 else 1)
                assert p.lo == max(0, p.z0 - 2) and p.hi == min(nz, p.z1 + 2)
                # owned lattice planes lie inside the exact region [2 lo + 1, 2 hi - 3] (or the box face)
                assert p.own_c0 >= (2 * p.lo + 1 if p.lo > 0 else 0)
                assert p.own_c1 - 1 <= (2 * p.hi - 3 if p.hi < nz else 2 * nz - 2)
                assert p.local_c0 == p.own_c0 - 2 * p.lo and p.local_c0 % 2 == 0
    assert mg.source_slice(10, 3, 0) == (0, 3) and mg.source_slice(10, 3, 2) == (6, 4)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        t = mg.HostTransport()
        # through the C function pointer, as msc3d_mg_compute calls it
        for n in (1, 8, 1000):
            send = (C.c_uint8 * n)(*[(rank * 7 + i) % 256 for i in range(n)])
            recv = (C.c_uint8 * (n * world))()
            assert t.struct.allgather(None, C.addressof(send), C.addressof(recv), n) == 0
            want = bytes((r * 7 + i) % 256 for r in range(world) for i in range(n))
            assert bytes(recv) == want
        assert t.calls == 3
        q.put((rank, True, ""))
    except Exception as e:  # pragma: no cover
        q.put((rank, False, repr(e)))
    finally:
        dist.destroy_process_group()


def _spawn(target, world, *args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=target, args=(r, world, port, q, *args)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=600) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    return res


def test_host_transport_gloo_world2():
    res = _spawn(_worker, 2)
    assert all(ok for _, ok, _ in res), res


def _slab_codes(values, dims, world):
    """Stitch the owned lattice planes of every slab's gradient (one GPU, in sequence)."""
    nx, ny, nz = dims
    ex, ey = 2 * nx - 1, 2 * ny - 1
    parts = []
    for r in range(world):
        plan = mg.slab_plan(nz, world, r)
        sv = mg.slab_values(values, dims, plan, own_only=False)
        ctx = m.Context(0)
        ctx.load_values(sv, (nx, ny, plan.local_nz)).gradient()
        local = ctx.get("codes")
        parts.append(local[plan.local_c0 * ex * ey:(plan.local_c0 + plan.own_c1 - plan.own_c0) * ex * ey])
        ctx.close()
    return np.concatenate(parts)


@pytest.mark.gpu
@pytest.mark.parametrize("kind,dims,world", [("gnoise", (24, 20, 16), 3), ("noise", (17, 13, 19), 4),
                                            ("gauss", (32, 32, 32), 2), ("gnoise", (64, 64, 64), 8)])
def test_slab_gradient_equals_whole(kind, dims, world):
    v = m.synth(kind, dims)
    ctx = m.Context(0)
    whole = ctx.load_values(v, dims).gradient() and ctx.get("codes")
    whole = ctx.get("codes")
    np.testing.assert_array_equal(_slab_codes(v, dims, world), whole)
    ctx.close()


@pytest.mark.gpu
@pytest.mark.parametrize("kind,dims,world", [("gnoise", (24, 20, 16), 3), ("noise", (20, 18, 16), 4),
                                            ("gnoise", (64, 64, 64), 8)])
def test_sharded_saddles_reassemble(kind, dims, world):
    import ctypes as C
    v = m.synth(kind, dims)
    want = m.compute(v, dims, with_segmentation=True)
    codes = _slab_codes(v, dims, world)
    blocks = {"src": [], "dst": [], "mult": []}
    ctx = m.Context(0)
    for r in range(world):
        ctx.load_codes(codes, dims)
        assert ctx._L.msc3d_ctx_compute_codes(ctx.h, m.OPT_SEGMENTATION, r, world, None) == 0
        for k in blocks:
            blocks[k].append(ctx.get("arcB_" + k))
        if r == 0:
            a = {k: ctx.get("arcA_" + k) for k in blocks}
            c = {k: ctx.get("arcC_" + k) for k in blocks}
            np.testing.assert_array_equal(ctx.get("cp_cell"), want.cp_cell)
            np.testing.assert_array_equal(ctx.get("labels_min"), want.labels_min)
            np.testing.assert_array_equal(ctx.get("labels_max"), want.labels_max)
    for k, w in (("src", want.arc_src), ("dst", want.arc_dst), ("mult", want.arc_mult)):
        got = np.concatenate([a[k]] + blocks[k] + [c[k]])
        np.testing.assert_array_equal(got, w)
    # one shard == the whole compute
    ctx.load_codes(codes, dims)
    assert ctx._L.msc3d_ctx_compute_codes(ctx.h, m.OPT_SEGMENTATION, 0, 1, None) == 0
    np.testing.assert_array_equal(ctx.get("arc_mult"), want.arc_mult)
    ctx.close()


def _mg_worker(rank, world, port, q, kind, dims, large_grid_path=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        v = m.synth(kind, dims)
        g = mg.MultiGPU(dims, rank, world, device=0, transport="host")
        if large_grid_path:  # what config 5 (> 2^32 cells) runs: scratch freed before the gather,
            for opt, val in (("release_transients", 1), ("term_rank_words", 1), ("frontier_cap", 16)):
                g.full.set_option(opt, val)  # (+ 2-saddle rank words, small frontiers: BFS rerun)
        own = torch.from_numpy(mg.slab_values(v, dims, g.plan)).cuda()
        for _ in range(2):  # a repeated step on the same contexts
            g.step(own, m.OPT_SEGMENTATION)
        got = g.outputs()
        want = m.compute(v, dims, with_segmentation=True)
        for k in ("cp_cell", "cp_index", "arc_src", "arc_dst", "arc_mult", "labels_min", "labels_max"):
            w = np.asarray(getattr(want, k))
            np.testing.assert_array_equal(got[k].view(w.dtype) if got[k].dtype != w.dtype else got[k], w,
                                          err_msg=k)
        assert g.transport.calls > 0
        g.close()
        q.put((rank, True, ""))
    except Exception as e:  # pragma: no cover
        import traceback
        q.put((rank, False, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("kind,dims,world", [("gnoise", (24, 20, 16), 2), ("noise", (20, 18, 17), 3),
                                            ("gauss", (40, 36, 32), 2)])
def test_mg_orchestrator_host_transport(kind, dims, world):
    res = _spawn(_mg_worker, world, kind, dims)
    assert all(ok for _, ok, _ in res), res


@pytest.mark.gpu
@pytest.mark.parametrize("kind,dims,world", [("gnoise", (24, 20, 16), 2), ("noise", (20, 18, 17), 3)])
def test_mg_orchestrator_large_grid_path(kind, dims, world):
    res = _spawn(_mg_worker, world, kind, dims, True)
    assert all(ok for _, ok, _ in res), res


@pytest.mark.gpu
def test_mg_orchestrator_nccl_world1():
    dims = (32, 28, 24)
    v = m.synth("gnoise", dims)
    g = mg.MultiGPU(dims, 0, 1, device=0, transport="nccl")
    own = torch.from_numpy(mg.slab_values(v, dims, g.plan)).cuda()
    g.step(own, m.OPT_SEGMENTATION)
    got = g.outputs()
    want = m.compute(v, dims, with_segmentation=True)
    for k in ("cp_cell", "arc_src", "arc_dst", "arc_mult", "labels_min", "labels_max"):
        np.testing.assert_array_equal(got[k], np.asarray(getattr(want, k)), err_msg=k)
    assert all(x >= 0 for x in g.stage_ms)
    g.close()

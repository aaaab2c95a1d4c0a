"""Multi-GPU decomposition (paper_2009_03707_b200/multigpu.py).

* CPU (gloo, world_size 2): slab plans, allgather-v, the code-plane gather.
* GPU (one device, shards run in sequence): z-slab gradients with 2-plane halos
  stitched into the whole GradientField equal the single-GPU codes byte for byte, and
  the 1-saddle-sharded saddle stages reassemble the single-GPU complex exactly.
"""
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
    for nz in (2, 3, 7, 16, 64, 512):
        for world in (1, 2, 3, 4, 8):
            if world > nz:
                continue
            plans = [mg.slab_plan(nz, world, r) for r in range(world)]
            assert plans[0].own_c0 == 0 and plans[-1].own_c1 == 2 * nz - 1
            for a, b in zip(plans, plans[1:]):
                assert a.own_c1 == b.own_c0 and a.z1 == b.z0
            for p in plans:
                assert p.lo <= max(0, p.z0 - 2) and p.hi >= min(nz, p.z1 + 2)
                # owned lattice planes lie inside the exact region [2 lo + 1, 2 hi - 3] (or the box face)
                assert p.own_c0 >= (2 * p.lo + 1 if p.lo > 0 else 0)
                assert p.own_c1 - 1 <= (2 * p.hi - 3 if p.hi < nz else 2 * nz - 2)
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
        # allgather-v of ragged blocks
        t = torch.arange(rank * 10, rank * 10 + 3 + 4 * rank, dtype=torch.int64)
        g = mg.allgather_v(t)
        want = torch.cat([torch.arange(r * 10, r * 10 + 3 + 4 * r) for r in range(world)])
        assert torch.equal(g, want)
        # code planes: rank r fills its slab grid's lattice with (global plane id + 1)
        nx, ny, nz = 3, 2, 7
        ex, ey = 2 * nx - 1, 2 * ny - 1
        plan = mg.slab_plan(nz, world, rank)
        local = torch.zeros((2 * plan.local_nz - 1) * ex * ey, dtype=torch.uint8)
        for lp in range(2 * plan.local_nz - 1):
            local[lp * ex * ey:(lp + 1) * ex * ey] = (lp + 2 * plan.lo + 1) % 256
        codes = mg.gather_codes(local, plan, ex * ey, mg.chunk_planes_for(nz, world))
        want = torch.repeat_interleave(torch.arange(1, 2 * nz, dtype=torch.uint8), ex * ey)
        assert torch.equal(codes, want)
        q.put((rank, True, ""))
    except Exception as e:  # pragma: no cover
        q.put((rank, False, repr(e)))
    finally:
        dist.destroy_process_group()


def test_collectives_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res), res


def _slab_codes(values, dims, world):
    """Stitch the owned lattice planes of every slab's gradient (one GPU, in sequence)."""
    nx, ny, nz = dims
    ex, ey = 2 * nx - 1, 2 * ny - 1
    parts = []
    for r in range(world):
        plan = mg.slab_plan(nz, world, r)
        sv = mg.slab_values(values, dims, plan)
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

"""bench.py -- MS complex throughput on B200 (BASELINE.json metric).

metric : end-to-end MS complex Mcells/s (N = (2nx-1)(2ny-1)(2nz-1) lattice cells per
         second) with per-stage ms vs the HBM roofline.
workload (N=1): BASELINE config 3 -- 512^3 float32 Gaussians + white noise, the
         north-star grid (dense critical points; saddle-saddle wavefront bottleneck).
step   : one full compute() (gradient, critical cells, extrema, reachability, path
         counting, device assembly incl. label volumes) over the resident grid.
value  : device-resident input, CUDA events on the pipeline stream, max over ranks.
e2e    : the same step through the public C ABI with HOST buffers: pinned input ->
         msc3d_ctx_load_values (H2D + validation) -> compute -> D2H of critical points,
         arcs and both label volumes.
--impl reference : the unmodified reference library (oracle/_ref, compiled from
         /root/reference) on the host cores, bounded sample of the same workload.
Multi-GPU: one process per GPU, each computing its own replica (weak scaling, no
data-path collective).
"""
import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "end-to-end MS complex Mcells/s and per-stage ms vs HBM roofline, 1/2/4/8 B200"
WORKLOAD = {"name": "config3_512cube_gnoise_f32", "dims": (512, 512, 512), "kind": "gnoise", "seed": 1}
CPU_SAMPLE = {"dims": (128, 128, 128), "kind": "gnoise", "seed": 1}
# like-for-like anchor: BASELINE config 2, small enough for the reference on the box's cores
PAIR = {"name": "config2_256cube_gauss_f32", "dims": (256, 256, 256), "kind": "gauss", "seed": 1}
STAGES = ("gradient", "critical", "extrema", "reachability", "counting")


def cells(d):
    return (2 * d[0] - 1) * (2 * d[1] - 1) * (2 * d[2] - 1)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        if args.impl != "reference":
            import torch
            # MSC3D_BENCH_BACKEND=gloo: development runs of several ranks on one GPU
            backend = os.environ.get("MSC3D_BENCH_BACKEND", "nccl")
            torch.cuda.set_device(local % torch.cuda.device_count())
            if backend == "nccl":
                dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
            else:
                dist.init_process_group(backend)
        else:
            dist.init_process_group("gloo")
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, world, device=None):
    if world <= 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def cpu_reference_run(sample, threads):
    """The unmodified reference compute() on the host; returns (seconds, timings, kind)."""
    import paper_2009_03707_b200 as m
    from oracle.pyoracle import REF_SO, Oracle64, Ref
    v = m.synth(sample["kind"], sample["dims"], sample["seed"]).astype(np.float64)
    if os.path.exists(REF_SO):
        r = Ref()
        out = r.compute(v, sample["dims"], threads=threads, with_segmentation=True)
        # compute()'s wall clock minus its serial field_hash (timed apart)
        return out["wall"] - out["hash_seconds"], list(out["timings"]), "reference", threads
    o = Oracle64()
    out = o.compute(v, sample["dims"])
    return out["wall"], None, "port", 1


def like_for_like(ctx, local, stream, reps=3):
    """BASELINE config 2 (256^3 gauss), both sides on this box: the GPU device-resident
    compute(), the GPU end to end through the C ABI with host buffers, the C++ drop-in
    msc3d::compute() (with and without the serial field_hash it overlaps), and the
    unmodified reference compute() on all host cores minus its field_hash (SURVEY.md
    8(d)); best of `reps` each."""
    import torch

    import paper_2009_03707_b200 as m
    from oracle.pyoracle import REF_SO, Ref
    if not os.path.exists(REF_SO):
        return None
    dims = PAIR["dims"]
    n = cells(dims)
    v = m.synth(PAIR["kind"], dims, PAIR["seed"])
    # GPU device-resident
    dev = torch.from_numpy(v).to(f"cuda:{local}")
    ctx.bind_values(dev.data_ptr(), dims, m.VALUE_F32)
    ctx.compute(m.OPT_SEGMENTATION)
    dev_ms = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        ctx.compute(m.OPT_SEGMENTATION)
        e1.record(stream)
        torch.cuda.synchronize()
        dev_ms.append(e0.elapsed_time(e1))
    # GPU end to end: pinned samples in, every output in pinned host memory
    c = [ctx.scalar(f"c{k}") for k in range(4)]
    na = ctx.scalar("arcs_min") + ctx.scalar("arcs_ss") + ctx.scalar("arcs_max")
    ncp, V = sum(c), dims[0] * dims[1] * dims[2]
    Cu = (dims[0] - 1) * (dims[1] - 1) * (dims[2] - 1)
    host_in = torch.from_numpy(v).pin_memory()
    b = {k: torch.empty(x, dtype=torch.uint8).pin_memory() for k, x in
         (("cp_cell", ncp * 4), ("cp_index", ncp), ("src", na * 4), ("dst", na * 4), ("mult", na * 8),
          ("lmin", V * 4), ("lmax", Cu * 4))}
    ho = m.HostOutputs(b["cp_cell"].data_ptr(), ncp * 4, b["cp_index"].data_ptr(), ncp, b["src"].data_ptr(),
                       b["dst"].data_ptr(), b["mult"].data_ptr(), na, b["lmin"].data_ptr(), b["lmax"].data_ptr(), 0, 0)
    e2e_s = []
    for _ in range(reps + 1):
        t0 = time.perf_counter()
        rc = ctx._L.msc3d_ctx_compute_host_values(ctx.h, m.Dims(*dims), m.VALUE_F32, C.c_void_p(host_in.data_ptr()),
                                                  m.OPT_SEGMENTATION, None, C.byref(ho))
        e2e_s.append(time.perf_counter() - t0)
        if rc:
            raise RuntimeError(f"compute_host failed: {rc}")
    # the C++ drop-in
    L = m.lib()
    L.msc3d_api_timed_compute.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int,
                                          C.POINTER(C.c_double)]
    out = (C.c_double * 8)()
    v32 = np.ascontiguousarray(v, dtype=np.float32)
    api, api_x = [], []
    for _ in range(reps + 1):
        if L.msc3d_api_timed_compute(v32.ctypes.data, dims[0], dims[1], dims[2], 1, out):
            raise RuntimeError("msc3d::compute() failed")
        api.append(out[0])
        api_x.append(out[6])
    # the unmodified reference on every host core
    threads = os.cpu_count() or 1
    r = Ref()
    ref_s, ref_stage = [], None
    v64 = v.astype(np.float64)
    for _ in range(reps):
        o = r.compute(v64, dims, threads=threads, with_segmentation=True)
        ref_s.append(o["wall"] - o["hash_seconds"])
        ref_stage = list(o["timings"])
    g_e2e, g_api, g_apix, cpu = min(e2e_s[1:]), min(api[1:]), min(api_x[1:]), min(ref_s)
    return {
        "workload": PAIR["name"], "dims": list(dims), "lattice_cells": n,
        "gpu_device_ms": min(dev_ms), "gpu_e2e_ms": g_e2e * 1e3, "gpu_api_ms": g_api * 1e3,
        "gpu_api_excl_field_hash_ms": g_apix * 1e3,
        "cpu_reference_ms": cpu * 1e3, "cpu_reference_stage_s": ref_stage, "cpu_cores": threads,
        "cpu_reference_field_hash_s": o["hash_seconds"],
        "speedup_e2e": cpu / g_e2e, "speedup_api_excl_field_hash": cpu / g_apix,
        "speedup_device": cpu / (min(dev_ms) / 1e3),
        "note": "same field and same box; reference = unmodified compute() on all host cores, wall minus its "
                "serial field_hash (SURVEY.md 8(d)); best of 3 each",
    }


def run_reference_arm(args, world, rank):
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    d = CPU_SAMPLE["dims"]
    times = []
    kind = "reference"
    used = threads
    for i in range(args.warmup + args.steps):
        secs, _, kind, used = cpu_reference_run(CPU_SAMPLE, threads)
        if i >= args.warmup:
            times.append(secs)
    t = sum(times) / len(times)
    val = cells(d) / t / 1e6
    sample = f"{d[0]}x{d[1]}x{d[2]} {CPU_SAMPLE['kind']} f32 (bounded sample of {WORKLOAD['name']}), full compute() with segmentation"
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "Mcells/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64-compare (f32 samples widened)",
        "data": "synthetic", "config": {"workload": WORKLOAD["name"], "sample": sample},
        "cpu_baseline": {"value": val, "unit": "Mcells/s", "cores": used, "kind": kind, "sample": sample},
        "e2e": {"value": val, "unit": "Mcells/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_sharded(args, world, rank, local):
    """N > 1: ONE grid across the ranks (strong scaling), orchestrated in C++
    (csrc/multigpu.cu, msc3d_mg_compute) over NCCL: P2P halo exchange + z-slab gradient,
    per-slab critical compaction (counts allgather, lists allgather-v), allgather-v of
    the owned code planes, extrema on the replicated codes, reachability + counting from
    each rank's 1-saddle slice, allgather-v of the arc blocks.  Every rank ends with the
    whole complex.  Each rank's input is its own vertex planes only."""
    import torch
    import torch.distributed as dist

    import paper_2009_03707_b200 as m
    from paper_2009_03707_b200 import multigpu as mg

    dims = WORKLOAD["dims"] if not args.size else (args.size,) * 3
    ncells = cells(dims)
    local = local % torch.cuda.device_count()
    transport = "host" if os.environ.get("MSC3D_BENCH_BACKEND", "nccl") != "nccl" else "nccl"
    g = mg.MultiGPU(dims, rank, world, device=local, transport=transport)
    v = m.synth(WORKLOAD["kind"], dims, WORKLOAD["seed"])  # every rank builds the same field
    sv = mg.slab_values(v, dims, g.plan)                    # ... and keeps its own planes
    dev_in = torch.from_numpy(sv).cuda()
    stream = torch.cuda.current_stream()
    g.set_stream(stream.cuda_stream)  # the step and the collectives on torch's stream
    for _ in range(args.warmup):
        g.step(dev_in, m.OPT_SEGMENTATION)
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    stage_acc = np.zeros(7)
    l0 = g.launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            stage_acc += np.array(g.step(dev_in, m.OPT_SEGMENTATION))
        ev1.record(stream)
        torch.cuda.synchronize()
    dist.barrier()
    ms_step = max_over_ranks(ev0.elapsed_time(ev1) / args.steps, world, f"cuda:{local}")
    value = ncells / (ms_step / 1e3) / 1e6
    launches = (g.launches() - l0) // args.steps
    n_arcs = int(g.full.array_info("arc_src")[1])
    if os.environ.get("MSC3D_BENCH_VERIFY") and rank == 0:
        # development check: the assembled complex equals the single-GPU compute()
        got = g.outputs()
        want = m.compute(v, dims, with_segmentation=True)
        for k in ("cp_cell", "arc_src", "arc_dst", "arc_mult", "labels_min", "labels_max"):
            if not np.array_equal(got[k], np.asarray(getattr(want, k))):
                raise AssertionError(f"sharded {k} differs from the single-GPU compute")
        print("verify ok: sharded complex == single-GPU compute", file=sys.stderr, flush=True)

    # e2e: host own planes in (pinned), step, rank 0 copies the assembled complex to host
    e2e = None
    if not args.no_e2e:
        host_in = torch.from_numpy(sv).pin_memory()
        outs = g.device_arrays()
        hbuf = {k: torch.empty(t.numel(), dtype=torch.uint8).pin_memory() for k, t in outs.items()
                if t is not None} if rank == 0 else {}
        times = []
        d2h = 0
        for i in range(2 + args.steps):
            torch.cuda.synchronize()
            dist.barrier()
            ta = time.perf_counter()
            dev_in.copy_(host_in, non_blocking=True)
            g.step(dev_in, m.OPT_SEGMENTATION)
            if rank == 0:  # the assembled complex to host: narrow arc arrays, decoded on host threads
                arrs = g.device_arrays()
                for k, t in arrs.items():
                    if t is not None and hbuf[k].numel() < t.numel():
                        hbuf[k] = torch.empty(t.numel(), dtype=torch.uint8).pin_memory()
                nb = {k: (t.numel() if t is not None else 0) for k, t in arrs.items()}
                ho = m.HostOutputs(hbuf["cp_cell"].data_ptr(), nb["cp_cell"], hbuf["cp_index"].data_ptr(),
                                   nb["cp_index"], hbuf["arc_src"].data_ptr(), hbuf["arc_dst"].data_ptr(),
                                   hbuf["arc_mult"].data_ptr(), nb["arc_src"] // 4,
                                   hbuf["labels_min"].data_ptr() if nb.get("labels_min") else 0,
                                   hbuf["labels_max"].data_ptr() if nb.get("labels_max") else 0, 0, 0)
                rc = g.full._L.msc3d_ctx_deliver_host(g.full.h, C.byref(ho))
                if rc:
                    raise RuntimeError(f"deliver_host failed: {rc}")
                d2h = g.full.scalar("d2h_bytes")
            torch.cuda.synchronize()
            tb = time.perf_counter()
            if i >= 2:
                times.append(tb - ta)
        te = max_over_ranks(sum(times) / len(times), world, f"cuda:{local}")
        e2e = {"value": ncells / te / 1e6, "unit": "Mcells/s", "ms_per_step": te * 1e3,
               "h2d_bytes_per_step": int(sv.nbytes), "d2h_bytes_per_step": int(d2h),
               "path": "per rank: pinned own planes -> device, msc3d_mg_compute (C++ + NCCL); "
                       "rank 0: complex -> pinned host (msc3d_ctx_deliver_host: narrow arc arrays)"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "Mcells/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": WORKLOAD["name"], "dims": list(dims), "field": WORKLOAD["kind"],
                       "seed": WORKLOAD["seed"], "lattice_cells": ncells,
                       "parallelism": f"z-slabs x{world} (P2P halos, gradient + critical) + allgather-v codes; "
                                      f"1-saddle shards x{world} (reachability, counting) + allgather-v arcs; "
                                      f"transport {transport}",
                       "l2": "inputs larger than L2"},
            "stages_ms_rank0": dict(zip(("halo+gradient", "critical+gathers", "extrema", "reachability",
                                         "counting", "arc_gather", "step"), (stage_acc / args.steps).tolist())),
            "e2e": e2e, "gpu_launches": int(launches), "counts": {"arcs": n_arcs},
            "clocks": clk.summary(), "cpu_baseline": None, "roofline": None,
        }
        print(json.dumps(line), flush=True)
    g.close()
    dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--size", type=int, default=0, help="dev only: cube size override")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-api", action="store_true", help="skip the C++ drop-in msc3d::compute() timing")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world, rank, local = dist_setup(args)
    if args.impl == "reference":
        return run_reference_arm(args, world, rank)
    if world > 1:
        return run_sharded(args, world, rank, local)

    import torch

    import paper_2009_03707_b200 as m

    torch.cuda.set_device(local)
    dims = WORKLOAD["dims"] if not args.size else (args.size,) * 3
    ncells = cells(dims)
    v = m.synth(WORKLOAD["kind"], dims, WORKLOAD["seed"])
    dev_in = torch.from_numpy(v).to(f"cuda:{local}")
    ctx = m.Context(local)
    stream = torch.cuda.Stream(device=local)
    ctx._L.msc3d_ctx_set_stream(ctx.h, C.c_void_p(stream.cuda_stream))
    torch.cuda.synchronize()
    ctx.bind_values(dev_in.data_ptr(), dims, m.VALUE_F32)

    for _ in range(args.warmup):
        ctx.compute(m.OPT_SEGMENTATION)
    torch.cuda.synchronize()

    # ---- timed region: device-resident input (inputs > L2: 512 MiB f32 + 1 GiB codes)
    stage_acc = np.zeros(5)
    l0 = ctx.launches()
    barrier(world)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(args.steps):
            ms = ctx.compute(m.OPT_SEGMENTATION)
            stage_acc += np.array(ms)
        ev1.record(stream)
        torch.cuda.synchronize()
    barrier(world)
    launches = (ctx.launches() - l0) // args.steps
    ms_step = ev0.elapsed_time(ev1) / args.steps
    ms_step = max_over_ranks(ms_step, world, f"cuda:{local}")
    value = world * ncells / (ms_step / 1e3) / 1e6
    stage_ms = (stage_acc / args.steps).tolist()

    # counts for the algorithmic-byte model
    c = [ctx.scalar(f"c{k}") for k in range(4)]
    a_min, a_ss, a_max = ctx.scalar("arcs_min"), ctx.scalar("arcs_ss"), ctx.scalar("arcs_max")
    V = dims[0] * dims[1] * dims[2]
    Cu = (dims[0] - 1) * (dims[1] - 1) * (dims[2] - 1)
    idb = 4 if ncells <= 0xFFFFFFFF else 8
    alg = {
        "gradient": 4 * V + ncells,
        "critical": ncells + idb * sum(c),
        "extrema": 5 * (V + Cu) + (12 if idb == 4 else 20) * (a_min + a_max),
        "reachability": ncells + ncells // 8,
        "counting": ncells + (16 if idb == 4 else 24) * a_ss,
    }
    peak, peak_kind = peaks()
    stages = {}
    for name, t in zip(STAGES, stage_ms):
        gbs = alg[name] / (t / 1e3) / 1e9 if t > 0 else 0.0
        stages[name] = {"ms": t, "alg_bytes": alg[name], "achieved_gbs": gbs, "frac": gbs / peak}
    dom = max(STAGES, key=lambda s: stages[s]["ms"])
    # DRAM traffic per stage from the committed ncu capture of the same workload
    # (tools/ncu_traffic.sh: dram__bytes_read.sum + dram__bytes_write.sum summed over
    # the stage's kernels of one compute()); None when absent
    traffic = {}
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        try:
            traffic = {k: v.get("dram_bytes") for k, v in json.load(open(tp)).items()}
        except Exception:
            traffic = {}
    for name in STAGES:
        stages[name]["dram_bytes_ncu"] = traffic.get(name)
        t = stages[name]["ms"]
        if traffic.get(name) and t > 0:  # what the stage actually moves through HBM
            stages[name]["dram_gbs_ncu"] = traffic[name] / (t / 1e3) / 1e9
            stages[name]["dram_frac_ncu"] = stages[name]["dram_gbs_ncu"] / peak
    roofline = {"bound": "hbm", "stage": dom, "achieved": stages[dom]["achieved_gbs"], "peak": peak,
                "peak_kind": peak_kind, "unit": "GB/s", "frac": stages[dom]["frac"],
                "traffic": traffic.get(dom), "alg_bytes_per_launch": alg[dom],
                "traffic_frac": stages[dom].get("dram_frac_ncu"),
                "note": "per stage (the reference's StageTimings unit): algorithmic bytes (SURVEY.md 8(d)) / "
                        "stage time from CUDA events on the pipeline stream; traffic = ncu DRAM bytes of the "
                        "stage's kernels for one compute() (profiles/traffic.json)"}

    # ---- e2e through the C ABI with host buffers: pinned f32 samples in, one
    # msc3d_ctx_compute_host_values call (upload in z-chunks overlapped with the
    # gradient, device validation, pipeline, every output copied to pinned host
    # buffers as soon as it is final); the wall clock covers all of it, every step.
    e2e = None
    if not args.no_e2e:
        host_in = torch.from_numpy(v).pin_memory()
        ncp = sum(c)
        n_arcs = a_min + a_ss + a_max
        idw = 4 if ncells <= 0xFFFFFFFF else 8
        V = dims[0] * dims[1] * dims[2]
        Cu = (dims[0] - 1) * (dims[1] - 1) * (dims[2] - 1)
        bufs = {
            "cp_cell": torch.empty(ncp * idw, dtype=torch.uint8).pin_memory(),
            "cp_index": torch.empty(ncp, dtype=torch.uint8).pin_memory(),
            "arc_src": torch.empty(n_arcs, dtype=torch.int32).pin_memory(),
            "arc_dst": torch.empty(n_arcs, dtype=torch.int32).pin_memory(),
            "arc_mult": torch.empty(n_arcs, dtype=torch.int64).pin_memory(),
            "labels_min": torch.empty(V, dtype=torch.int32).pin_memory(),
            "labels_max": torch.empty(Cu, dtype=torch.int32).pin_memory(),
        }
        ho = m.HostOutputs(bufs["cp_cell"].data_ptr(), ncp * idw, bufs["cp_index"].data_ptr(), ncp,
                           bufs["arc_src"].data_ptr(), bufs["arc_dst"].data_ptr(), bufs["arc_mult"].data_ptr(),
                           n_arcs, bufs["labels_min"].data_ptr(), bufs["labels_max"].data_ptr(), 0, 0)
        e2e_times = []
        h2d = V * 4
        d2h = 0
        for i in range(2 + args.steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            rc = ctx._L.msc3d_ctx_compute_host_values(ctx.h, m.Dims(*dims), m.VALUE_F32,
                                                      C.c_void_p(host_in.data_ptr()), m.OPT_SEGMENTATION, None,
                                                      C.byref(ho))
            t1 = time.perf_counter()
            if rc:
                raise RuntimeError(f"compute_host failed: {rc}")
            d2h = ctx.scalar("d2h_bytes")  # as counted by the delivery (multiplicities as bytes + escapes)
            if i >= 2:
                e2e_times.append(t1 - t0)
        if ho.n_arcs != n_arcs or ho.n_cp != ncp:
            raise RuntimeError("e2e output sizes differ from the device-resident run")
        te = max_over_ranks(sum(e2e_times) / len(e2e_times), world, f"cuda:{local}")
        e2e = {"value": world * ncells / te / 1e6, "unit": "Mcells/s", "ms_per_step": te * 1e3,
               "step_ms": [round(x * 1e3, 1) for x in e2e_times],
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": int(d2h),
               "path": "msc3d_ctx_compute_host_values (C ABI): pinned samples in (upload overlapped with the "
                       "gradient), pinned host outputs (copies overlapped with the later stages; multiplicities "
                       "as one byte per arc + escapes, widened into the u64 output by host threads)"}

    # ---- the C++ drop-in msc3d::compute() (include/msc3d/api.hpp): host ScalarField of
    # doubles in, host MSComplex out (critical points with coordinates and values,
    # Arc vector, label volumes, input_hash) -- what a reference user's call costs.
    # One warm-up call (pins the staging buffers), one timed; field_hash alone beside.
    api = None
    if rank == 0 and world == 1 and not args.no_api:
        L = m.lib()
        L.msc3d_api_timed_compute.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int,
                                              C.POINTER(C.c_double)]
        out = (C.c_double * 8)()
        v32 = np.ascontiguousarray(v, dtype=np.float32)
        secs = []
        for _ in range(2):
            rc = L.msc3d_api_timed_compute(v32.ctypes.data, dims[0], dims[1], dims[2], 1, out)
            if rc:
                raise RuntimeError(f"msc3d::compute() failed: {rc}")
            secs.append(out[0])
        if int(out[2]) != a_min + a_ss + a_max or int(out[1]) != sum(c):
            raise RuntimeError("msc3d::compute() output sizes differ from the device-resident run")
        api = {"value": ncells / secs[-1] / 1e6, "unit": "Mcells/s", "seconds": secs[-1],
               "first_call_seconds": secs[0], "field_hash_seconds": out[3],
               "seconds_excl_field_hash": out[6], "value_excl_field_hash": ncells / out[6] / 1e6,
               "path": "msc3d::compute(ScalarField, {with_segmentation}) -> MSComplex (C++ drop-in API): "
                       "parallel f32 conversion + pinned upload, device pipeline, pinned download, parallel "
                       "host assembly; the byte-serial field_hash (FNV-1a, msc.cpp:31-42) runs concurrently"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        secs, tim, kind, used = cpu_reference_run(CPU_SAMPLE, threads)
        d = CPU_SAMPLE["dims"]
        cpu = {"value": cells(d) / secs / 1e6, "unit": "Mcells/s", "cores": used, "kind": kind,
               "sample": f"{d[0]}^3 {CPU_SAMPLE['kind']} f32, one full compute() with segmentation, "
                         f"threads={used}", "seconds": secs, "stage_s": tim}

    pair = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not args.size:
        pair = like_for_like(ctx, local, stream)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "Mcells/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": WORKLOAD["name"], "dims": list(dims), "field": WORKLOAD["kind"],
                       "seed": WORKLOAD["seed"], "lattice_cells": ncells,
                       "parallelism": f"replicas x{world}", "l2": "inputs larger than L2 (512 MiB f32 in, 1 GiB codes)"},
            "stages_ms": dict(zip(STAGES, stage_ms)), "stages": stages, "roofline": roofline,
            "cpu_baseline": cpu, "e2e": e2e, "e2e_api": api, "like_for_like": pair, "gpu_launches": int(launches),
            "counts": {"critical": c, "arcs_min": a_min, "arcs_ss": a_ss, "arcs_max": a_max},
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

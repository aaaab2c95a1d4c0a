// Multi-GPU MS complex, host orchestration in C++ (BASELINE.json
// north_star: "the grid is slab-partitioned with one-layer halos exchanged by P2P/NCCL
// over NVLink for the gradient and critical-point stages ... the arcs are gathered
// with NCCL allgather-v").  The reference has no counterpart: its only parallelism is
// the host thread pool of primitives.cpp:9-42.
//
// One process per GPU.  A step on rank r of G (plan: msc3d_mg_plan):
//   1. halo exchange: the rank holds its own vertex planes [z0, z1); it sends its first
//      / last kHalo planes to rank r-1 / r+1 and receives theirs (ncclSend/ncclRecv in
//      one group) into the slab grid [lo, hi) = [z0 - 2, z1 + 2) clipped to the box;
//   2. gradient of the slab grid (gradient.cpp:79-283): a lower star lies in the 3x3x3
//      neighbourhood of its vertex (gradient.cpp:13-20), so every cell of the rank's own
//      lattice planes [2 z0, 2 z1) gets its exact code (vertex ids are shifted on the
//      slab, which the tie-break tolerates: it only compares ids, the shift keeps
//      their order);
//   3. critical cells of the owned planes (gradient.cpp:285-297): the same bit-parallel
//      compaction over that plane range, ids shifted to global cell ids; the global
//      lists are the per-slab lists concatenated in rank (= z = id) order -- counts by
//      an allgather, lists by an allgather-v;
//   4. allgather-v of the owned code planes: every rank holds the whole GradientField
//      (the north star's replicated gradient field);
//   5. extrema on the replicated codes (replicated), reachability + path counting from
//      the rank's balanced slice of the critical 1-cells (a z-slab of sources: its
//      1s->2s arcs are a contiguous block of the global sorted arc list);
//   6. allgather-v of the arc blocks; min->1s ∥ blocks in rank order ∥ 2s->max.
// Every rank ends with the whole complex in its full-grid context ("cp_cell",
// "cp_index", "arc_src/dst/mult", "labels_min/max") -- identical to a single-GPU
// compute() (tests/test_multigpu.py).
//
// Transports (msc3d_comm): NCCL (libnccl.so.2 resolved at run time with dlopen -- the
// same library torch.distributed loads -- no link-time dependency), or host callbacks
// (an allgather over host buffers, e.g. torch.distributed/gloo: several ranks sharing
// one GPU in the tests).  Collectives run on the full-grid context's stream.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "ctx.cuh"
#include "stages.cuh"

namespace {

// failures name the orchestrator line on stderr (a rank's error otherwise only shows
// up as its peers' broken collectives)
#define TRY(x)                                                                             \
    do {                                                                                   \
        const int _rc = (x);                                                               \
        if (_rc != MSC3D_OK) {                                                             \
            std::fprintf(stderr, "msc3d multigpu.cu:%d: status %d (%s)\n", __LINE__, _rc, #x); \
            return _rc;                                                                    \
        }                                                                                  \
    } while (0)

constexpr int kHalo = 2;  // vertex planes of halo on each side of a slab

// ---- NCCL through dlopen -------------------------------------------------------------
struct Nccl {
    void* lib = nullptr;
    bool tried = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;

    bool load() {
        if (tried) return lib != nullptr;
        tried = true;
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            lib = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (lib) break;
        }
        if (!lib) return false;
        auto sym = [&](auto& fn, const char* s) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(lib, s));
            return fn != nullptr;
        };
        const bool ok = sym(GetUniqueId, "ncclGetUniqueId") && sym(CommInitRank, "ncclCommInitRank") &&
                        sym(CommDestroy, "ncclCommDestroy") && sym(AllGather, "ncclAllGather") &&
                        sym(Broadcast, "ncclBroadcast") && sym(Send, "ncclSend") && sym(Recv, "ncclRecv") &&
                        sym(GroupStart, "ncclGroupStart") && sym(GroupEnd, "ncclGroupEnd");
        if (!ok) lib = nullptr;
        return lib != nullptr;
    }
};
Nccl g_nccl;

#define NCCL_TRY(x)                                        \
    do {                                                   \
        if ((x) != ncclSuccess) return MSC3D_ERR_CUDA;     \
    } while (0)

// ---- slab plan ------------------------------------------------------------------------
struct Plan {
    std::int64_t z0, z1, lo, hi, own_c0, own_c1, local_c0;
};
Plan plan_of(std::int64_t nz, int world, int rank) {
    Plan p;
    p.z0 = nz * rank / world;
    p.z1 = nz * (rank + 1) / world;
    p.lo = std::max<std::int64_t>(0, p.z0 - kHalo);
    p.hi = std::min<std::int64_t>(nz, p.z1 + kHalo);
    p.own_c0 = 2 * p.z0;
    p.own_c1 = rank == world - 1 ? 2 * nz - 1 : 2 * p.z1;
    p.local_c0 = p.own_c0 - 2 * p.lo;
    return p;
}

__global__ void k_add_offset(void* ids, std::uint64_t n, int width, std::uint64_t off) {
    for (std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<std::uint64_t>(gridDim.x) * blockDim.x) {
        if (width == 4) static_cast<std::uint32_t*>(ids)[i] += static_cast<std::uint32_t>(off);
        else static_cast<std::uint64_t*>(ids)[i] += off;
    }
}

}  // namespace

struct msc3d_comm {
    int rank = 0, world = 1;
    ncclComm_t nccl = nullptr;
    msc3d_host_transport host{};
    bool use_nccl = false;

    // every rank contributes `bytes` from device `send`; device `recv` gets world*bytes
    int allgather(const void* send, void* recv, std::uint64_t bytes, cudaStream_t s) {
        if (use_nccl) {
            NCCL_TRY(g_nccl.AllGather(send, recv, bytes, ncclUint8, nccl, s));
            return MSC3D_OK;
        }
        std::vector<std::uint8_t> hs(bytes), hr(bytes * world);
        if (bytes) MSC3D_CUDA_TRY(cudaMemcpyAsync(hs.data(), send, bytes, cudaMemcpyDeviceToHost, s));
        MSC3D_CUDA_TRY(cudaStreamSynchronize(s));
        if (host.allgather(host.user, hs.data(), hr.data(), bytes) != 0) return MSC3D_ERR_RUNTIME;
        if (bytes) MSC3D_CUDA_TRY(cudaMemcpyAsync(recv, hr.data(), bytes * world, cudaMemcpyHostToDevice, s));
        MSC3D_CUDA_TRY(cudaStreamSynchronize(s));
        return MSC3D_OK;
    }
    // host values: every rank's u64 vector of length n, concatenated in rank order
    int allgather_u64(const std::vector<std::uint64_t>& mine, std::vector<std::uint64_t>& all, msc3d_ctx* ctx) {
        const std::uint64_t n = mine.size();
        all.assign(n * world, 0);
        if (!use_nccl)
            return host.allgather(host.user, mine.data(), all.data(), n * 8) == 0 ? MSC3D_OK : MSC3D_ERR_RUNTIME;
        auto* d = static_cast<std::uint64_t*>(ctx->ensure("mg_u64", n * (world + 1), 8));
        if (!d) return MSC3D_ERR_NOMEM;
        MSC3D_CUDA_TRY(cudaMemcpyAsync(d, mine.data(), n * 8, cudaMemcpyHostToDevice, ctx->stream));
        TRY(allgather(d, d + n, n * 8, ctx->stream));
        MSC3D_CUDA_TRY(cudaMemcpyAsync(all.data(), d + n, n * world * 8, cudaMemcpyDeviceToHost, ctx->stream));
        MSC3D_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
        return MSC3D_OK;
    }
    // allgather-v with known sizes: rank q's sizes[q] bytes land at recv + offset[q]
    // (exact, no padding: one ncclBroadcast per root inside a group)
    int allgather_v(const void* send, void* recv, const std::vector<std::uint64_t>& sizes, cudaStream_t s) {
        std::vector<std::uint64_t> off(world + 1, 0);
        for (int q = 0; q < world; ++q) off[q + 1] = off[q] + sizes[q];
        auto* out = static_cast<std::uint8_t*>(recv);
        if (use_nccl) {
            NCCL_TRY(g_nccl.GroupStart());
            for (int q = 0; q < world; ++q)
                if (sizes[q])
                    NCCL_TRY(g_nccl.Broadcast(q == rank ? send : nullptr, out + off[q], sizes[q], ncclUint8, q, nccl, s));
            NCCL_TRY(g_nccl.GroupEnd());
            return MSC3D_OK;
        }
        // host transport: one padded allgather
        const std::uint64_t m = *std::max_element(sizes.begin(), sizes.end());
        std::vector<std::uint8_t> hs(m, 0), hr(m * world);
        if (sizes[rank]) MSC3D_CUDA_TRY(cudaMemcpyAsync(hs.data(), send, sizes[rank], cudaMemcpyDeviceToHost, s));
        MSC3D_CUDA_TRY(cudaStreamSynchronize(s));
        if (host.allgather(host.user, hs.data(), hr.data(), m) != 0) return MSC3D_ERR_RUNTIME;
        for (int q = 0; q < world; ++q)
            if (sizes[q]) MSC3D_CUDA_TRY(cudaMemcpyAsync(out + off[q], hr.data() + q * m, sizes[q], cudaMemcpyHostToDevice, s));
        MSC3D_CUDA_TRY(cudaStreamSynchronize(s));
        return MSC3D_OK;
    }
    // halo exchange over device buffers: send_lo -> rank-1, send_hi -> rank+1;
    // recv_lo <- rank-1 (its send_hi), recv_hi <- rank+1 (its send_lo); all `bytes` long
    int halo(const void* send_lo, const void* send_hi, void* recv_lo, void* recv_hi, std::uint64_t bytes,
             cudaStream_t s) {
        if (world == 1 || bytes == 0) return MSC3D_OK;
        if (use_nccl) {  // P2P over NVLink
            NCCL_TRY(g_nccl.GroupStart());
            if (rank > 0) {
                NCCL_TRY(g_nccl.Send(send_lo, bytes, ncclUint8, rank - 1, nccl, s));
                NCCL_TRY(g_nccl.Recv(recv_lo, bytes, ncclUint8, rank - 1, nccl, s));
            }
            if (rank < world - 1) {
                NCCL_TRY(g_nccl.Send(send_hi, bytes, ncclUint8, rank + 1, nccl, s));
                NCCL_TRY(g_nccl.Recv(recv_hi, bytes, ncclUint8, rank + 1, nccl, s));
            }
            NCCL_TRY(g_nccl.GroupEnd());
            return MSC3D_OK;
        }
        // host transport: every rank publishes both boundary blocks; neighbours pick theirs
        std::vector<std::uint8_t> hs(2 * bytes, 0), hr(2 * bytes * world);
        MSC3D_CUDA_TRY(cudaMemcpyAsync(hs.data(), send_lo, bytes, cudaMemcpyDeviceToHost, s));
        MSC3D_CUDA_TRY(cudaMemcpyAsync(hs.data() + bytes, send_hi, bytes, cudaMemcpyDeviceToHost, s));
        MSC3D_CUDA_TRY(cudaStreamSynchronize(s));
        if (host.allgather(host.user, hs.data(), hr.data(), 2 * bytes) != 0) return MSC3D_ERR_RUNTIME;
        if (rank > 0)
            MSC3D_CUDA_TRY(cudaMemcpyAsync(recv_lo, hr.data() + (rank - 1) * 2 * bytes + bytes, bytes,
                                           cudaMemcpyHostToDevice, s));
        if (rank < world - 1)
            MSC3D_CUDA_TRY(cudaMemcpyAsync(recv_hi, hr.data() + (rank + 1) * 2 * bytes, bytes, cudaMemcpyHostToDevice, s));
        MSC3D_CUDA_TRY(cudaStreamSynchronize(s));
        return MSC3D_OK;
    }
};

struct msc3d_mg {
    msc3d_comm* comm = nullptr;
    msc3d_ctx* slab = nullptr;  // the slab grid (own planes + halos)
    msc3d_ctx* full = nullptr;  // the whole grid (replicated codes, sharded saddle stages)
    std::uint64_t launches0 = 0;
};

namespace {

int ctx_new(int device, msc3d_ctx** out) { return msc3d_ctx_create(out, device); }

// Critical cells of lattice planes [c0, c1) of the slab context's codes, as global ids
// (offset `shift` cells) of width w, into the slab context's "mg_crit0..3".
int slab_critical(msc3d_ctx* ctx, std::int64_t c0, std::int64_t c1, int w, std::uint64_t shift,
                  std::uint64_t counts[4]) {
    using msc3d_dev::Dims;
    const Dims& d = ctx->dims;
    Dims sub = Dims::make(d.nx, d.ny, (c1 - c0) / 2 + 1);  // ex, ey, parity of planes preserved (c0 even)
    sub.n_cells = static_cast<std::uint64_t>(c1 - c0) * d.exy;
    // the owned planes as their own (aligned) array: the compaction kernels read 16-byte
    // vectors; it is also this rank's block of the code allgather
    auto* codes = static_cast<std::uint8_t*>(ctx->ensure("mg_own_codes", sub.n_cells, 1));
    if (!codes) return MSC3D_ERR_NOMEM;
    MSC3D_CUDA_TRY(cudaMemcpyAsync(codes, ctx->ptr<std::uint8_t>("codes") + static_cast<std::uint64_t>(c0) * d.exy,
                                   sub.n_cells, cudaMemcpyDeviceToDevice, ctx->stream));
    TRY(msc3d_dev::launch_critical_count(codes, sub, ctx->d_small, ctx->stream, ctx->num_sms));
    TRY(ctx->fetch_small(4));
    void* outs[4];
    for (int k = 0; k < 4; ++k) {
        counts[k] = ctx->h_small[k];
        outs[k] = ctx->ensure("mg_crit" + std::to_string(k), counts[k], w);
        if (!outs[k]) return MSC3D_ERR_NOMEM;
    }
    TRY(msc3d_dev::launch_critical_compact(codes, sub, ctx->ws, outs, w, ctx->d_small + 8, ctx->stream));
    for (int k = 0; k < 4; ++k)
        if (counts[k] && shift) {
            const unsigned grid = static_cast<unsigned>(std::min<std::uint64_t>((counts[k] + 255) / 256, 4096));
            k_add_offset<<<grid, 256, 0, ctx->stream>>>(outs[k], counts[k], w, shift);
            msc3d_dev::count_launch();
        }
    MSC3D_CUDA_TRY(cudaGetLastError());
    return MSC3D_OK;
}

double elapsed(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return ms;
}

}  // namespace

extern "C" {

int msc3d_mg_plan(int64_t nz, int world, int rank, int64_t out[7]) {
    if (world < 1 || rank < 0 || rank >= world || nz < 2) return MSC3D_ERR_INVALID;
    const Plan p = plan_of(nz, world, rank);
    const int64_t v[7] = {p.z0, p.z1, p.lo, p.hi, p.own_c0, p.own_c1, p.local_c0};
    std::memcpy(out, v, sizeof v);
    // the halo comes from the neighbours' own planes: each rank must own >= kHalo
    return (world > 1 && nz / world < kHalo) ? MSC3D_ERR_INVALID : MSC3D_OK;
}

int msc3d_nccl_unique_id(uint8_t out[128]) {
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    if (!g_nccl.load()) return MSC3D_ERR_STATE;
    ncclUniqueId id;
    NCCL_TRY(g_nccl.GetUniqueId(&id));
    std::memcpy(out, &id, sizeof id);
    return MSC3D_OK;
}

int msc3d_comm_create_nccl(msc3d_comm** out, const uint8_t id[128], int rank, int world, int device) {
    *out = nullptr;
    if (world < 1 || rank < 0 || rank >= world) return MSC3D_ERR_INVALID;
    if (!g_nccl.load()) return MSC3D_ERR_STATE;
    MSC3D_CUDA_TRY(cudaSetDevice(device));
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof uid);
    auto* c = new msc3d_comm();
    c->rank = rank;
    c->world = world;
    c->use_nccl = true;
    if (g_nccl.CommInitRank(&c->nccl, world, uid, rank) != ncclSuccess) {
        delete c;
        return MSC3D_ERR_CUDA;
    }
    *out = c;
    return MSC3D_OK;
}

int msc3d_comm_create_host(msc3d_comm** out, const msc3d_host_transport* t, int rank, int world) {
    *out = nullptr;
    if (!t || !t->allgather || world < 1 || rank < 0 || rank >= world) return MSC3D_ERR_INVALID;
    auto* c = new msc3d_comm();
    c->rank = rank;
    c->world = world;
    c->host = *t;
    *out = c;
    return MSC3D_OK;
}

void msc3d_comm_destroy(msc3d_comm* c) {
    if (!c) return;
    if (c->nccl && g_nccl.CommDestroy) g_nccl.CommDestroy(c->nccl);
    delete c;
}

int msc3d_mg_create(msc3d_mg** out, msc3d_comm* comm, int device) {
    *out = nullptr;
    if (!comm) return MSC3D_ERR_INVALID;
    auto* g = new msc3d_mg();
    g->comm = comm;
    int rc = ctx_new(device, &g->slab);
    if (rc == MSC3D_OK) rc = ctx_new(device, &g->full);
    if (rc != MSC3D_OK) {
        if (g->slab) msc3d_ctx_destroy(g->slab);
        delete g;
        return rc;
    }
    // one stream for both contexts and the collectives
    msc3d_ctx_set_stream(g->slab, g->full->stream);
    g->slab->own_stream = false;
    *out = g;
    return MSC3D_OK;
}

void msc3d_mg_destroy(msc3d_mg* g) {
    if (!g) return;
    msc3d_ctx_destroy(g->slab);
    msc3d_ctx_destroy(g->full);
    delete g;
}

msc3d_ctx* msc3d_mg_full_ctx(msc3d_mg* g) { return g->full; }
msc3d_ctx* msc3d_mg_slab_ctx(msc3d_mg* g) { return g->slab; }

int msc3d_mg_set_stream(msc3d_mg* g, void* stream) {
    if (!stream) return MSC3D_OK;
    TRY(msc3d_ctx_set_stream(g->full, stream));
    return msc3d_ctx_set_stream(g->slab, stream);
}

int msc3d_mg_compute(msc3d_mg* g, msc3d_dims dims, int value_type, const void* own_values, int options,
                     double* stage_ms) {
    msc3d_comm* cm = g->comm;
    msc3d_ctx* full = g->full;
    msc3d_ctx* slab = g->slab;
    const cudaStream_t s = full->stream;
    const int world = cm->world, rank = cm->rank;
    int64_t pv[7];
    TRY(msc3d_mg_plan(dims.nz, world, rank, pv));
    const Plan p = plan_of(dims.nz, world, rank);
    if (value_type != MSC3D_VALUE_F32 && value_type != MSC3D_VALUE_F64) return MSC3D_ERR_INVALID;
    const std::uint64_t esz = value_type == MSC3D_VALUE_F64 ? 8 : 4;
    const std::uint64_t plane = static_cast<std::uint64_t>(dims.nx) * dims.ny;
    cudaEvent_t ev[8] = {};
    for (auto& e : ev) cudaEventCreate(&e);
    struct Guard {
        cudaEvent_t* e;
        ~Guard() {
            for (int i = 0; i < 8; ++i)
                if (e[i]) cudaEventDestroy(e[i]);
        }
    } guard{ev};
    cudaEventRecord(ev[0], s);

    // [1] halo exchange into the slab grid [lo, hi)
    const std::uint64_t nslab = static_cast<std::uint64_t>(p.hi - p.lo) * plane;
    auto* sv = static_cast<std::uint8_t*>(slab->ensure("mg_slab_values", nslab, static_cast<int>(esz)));
    if (!sv) return MSC3D_ERR_NOMEM;
    const std::uint64_t own_bytes = static_cast<std::uint64_t>(p.z1 - p.z0) * plane * esz;
    MSC3D_CUDA_TRY(cudaMemcpyAsync(sv + (p.z0 - p.lo) * plane * esz, own_values, own_bytes, cudaMemcpyDeviceToDevice, s));
    {
        const std::uint64_t hb = kHalo * plane * esz;
        const auto* own = static_cast<const std::uint8_t*>(own_values);
        TRY(cm->halo(own, own + own_bytes - hb, sv, sv + (p.z1 - p.lo) * plane * esz, hb, s));
    }
    // [2] gradient of the slab grid
    msc3d_dims sd{dims.nx, dims.ny, p.hi - p.lo};
    TRY(msc3d_ctx_bind_values(slab, sd, value_type, sv));
    TRY(msc3d_stage::gradient(slab, false));
    cudaEventRecord(ev[1], s);

    // [3] critical cells of the owned planes, global ids; counts then lists gathered
    const msc3d_dims gd{dims.nx, dims.ny, dims.nz};
    {  // the full context's grid (id width from the whole lattice)
        full->dims = msc3d_dev::Dims::make(dims.nx, dims.ny, dims.nz);
        full->have_dims = true;
    }
    const int w = full->id_width();
    const std::uint64_t exy = static_cast<std::uint64_t>(full->dims.exy);
    std::uint64_t cnt[4];
    TRY(slab_critical(slab, p.local_c0, p.local_c0 + (p.own_c1 - p.own_c0), w,
                      static_cast<std::uint64_t>(p.own_c0) * exy, cnt));
    std::vector<std::uint64_t> all;
    TRY(cm->allgather_u64(std::vector<std::uint64_t>(cnt, cnt + 4), all, full));
    for (int k = 0; k < 4; ++k) {
        std::vector<std::uint64_t> sizes(world);
        std::uint64_t tot = 0;
        for (int q = 0; q < world; ++q) {
            sizes[q] = all[4 * q + k] * w;
            tot += all[4 * q + k];
        }
        void* dst = full->ensure("crit" + std::to_string(k), tot, w);
        if (!dst) return MSC3D_ERR_NOMEM;
        TRY(cm->allgather_v(slab->ptr<void>("mg_crit" + std::to_string(k)), dst, sizes, s));
        full->scalars["c" + std::to_string(k)] = static_cast<std::int64_t>(tot);
    }
    // [4] the replicated GradientField: owned code planes of every rank
    {
        auto* codes = full->ensure("codes", full->dims.n_cells, 1);
        if (!codes) return MSC3D_ERR_NOMEM;
        std::vector<std::uint64_t> sizes(world);
        for (int q = 0; q < world; ++q) {
            const Plan pq = plan_of(dims.nz, world, q);
            sizes[q] = static_cast<std::uint64_t>(pq.own_c1 - pq.own_c0) * exy;
        }
        TRY(cm->allgather_v(slab->ptr<std::uint8_t>("mg_own_codes"), codes, sizes, s));
        full->crit_counts_valid = false;
    }
    full->values = nullptr;  // only codes travel; cp values need the samples (not gathered)
    full->crit_external = true;
    cudaEventRecord(ev[2], s);

    // [5] extrema (replicated) + reachability / counting from this rank's 1-saddle slice
    double st[5] = {0, 0, 0, 0, 0};
    TRY(msc3d_stage::compute_from_codes(full, options, st, nullptr, false, static_cast<std::uint64_t>(rank),
                                        static_cast<std::uint64_t>(world), nullptr, true));
    cudaEventRecord(ev[3], s);

    // [6] the arc blocks of every rank, then min->1s ∥ blocks ∥ 2s->max.  On grids
    // above 2^32 cells the saddle stages' scratch goes first (config 5: ~25 GB of
    // junction records, pools and frontiers make room for the gathered arcs).
    if (world > 1 && full->release_transients())
        for (const char* t : {"frontier_a", "frontier_b", "heavy_q", "indeg", "jbits", "jcount", "jdest", "jfwd",
                              "jlist", "jnode", "joff", "jrank", "jrec", "ovoff", "pending", "pending0", "pool_cnt",
                              "pool_key", "ready0", "soff", "term_rank", "tmap", "visited", "slen", "rsrc",
                              "ready_bits", "jump_conv_pt", "predone", "ptbits", "count_stats"})
            full->release(t);
    if (world > 1) {
        const std::uint64_t na = full->count("arcA_src"), nb = full->count("arcB_src"), nc = full->count("arcC_src");
        std::vector<std::uint64_t> allnb;
        TRY(cm->allgather_u64({nb}, allnb, full));
        std::uint64_t tb = 0;
        for (auto x : allnb) tb += x;
        const std::uint64_t total = na + tb + nc;
        auto* asrc = static_cast<std::uint32_t*>(full->ensure("arc_src", total, 4));
        auto* adst = static_cast<std::uint32_t*>(full->ensure("arc_dst", total, 4));
        auto* amul = static_cast<std::uint64_t*>(full->ensure("arc_mult", total, 8));
        if (!asrc || !adst || !amul) return MSC3D_ERR_NOMEM;
        std::vector<std::uint64_t> s4(world), s8(world);
        for (int q = 0; q < world; ++q) {
            s4[q] = allnb[q] * 4;
            s8[q] = allnb[q] * 8;
        }
        TRY(cm->allgather_v(full->ptr<void>("arcB_src"), asrc + na, s4, s));
        TRY(cm->allgather_v(full->ptr<void>("arcB_dst"), adst + na, s4, s));
        TRY(cm->allgather_v(full->ptr<void>("arcB_mult"), amul + na, s8, s));
        if (na) {
            MSC3D_CUDA_TRY(cudaMemcpyAsync(asrc, full->ptr<void>("arcA_src"), na * 4, cudaMemcpyDeviceToDevice, s));
            MSC3D_CUDA_TRY(cudaMemcpyAsync(adst, full->ptr<void>("arcA_dst"), na * 4, cudaMemcpyDeviceToDevice, s));
            MSC3D_CUDA_TRY(cudaMemcpyAsync(amul, full->ptr<void>("arcA_mult"), na * 8, cudaMemcpyDeviceToDevice, s));
        }
        if (nc) {
            MSC3D_CUDA_TRY(cudaMemcpyAsync(asrc + na + tb, full->ptr<void>("arcC_src"), nc * 4, cudaMemcpyDeviceToDevice, s));
            MSC3D_CUDA_TRY(cudaMemcpyAsync(adst + na + tb, full->ptr<void>("arcC_dst"), nc * 4, cudaMemcpyDeviceToDevice, s));
            MSC3D_CUDA_TRY(cudaMemcpyAsync(amul + na + tb, full->ptr<void>("arcC_mult"), nc * 8, cudaMemcpyDeviceToDevice, s));
        }
        full->scalars["arcs_total"] = static_cast<std::int64_t>(total);
        if (full->release_transients()) {  // the blocks now live in arc_src/dst/mult
            MSC3D_CUDA_TRY(cudaStreamSynchronize(s));
            for (const char* t : {"arcA_src", "arcA_dst", "arcA_mult", "arcB_src", "arcB_dst", "arcB_mult",
                                  "arcC_src", "arcC_dst", "arcC_mult"})
                full->release(t);
        }
    }
    cudaEventRecord(ev[4], s);
    MSC3D_CUDA_TRY(cudaStreamSynchronize(s));
    if (stage_ms) {
        // [0] halo + slab gradient [1] slab critical + gathers of lists and codes
        // [2] extrema [3] reachability [4] counting [5] arc gather [6] whole step
        stage_ms[0] = elapsed(ev[0], ev[1]);
        stage_ms[1] = elapsed(ev[1], ev[2]);
        stage_ms[2] = st[2];
        stage_ms[3] = st[3];
        stage_ms[4] = st[4];
        stage_ms[5] = elapsed(ev[3], ev[4]);
        stage_ms[6] = elapsed(ev[0], ev[4]);
    }
    (void)gd;
    return MSC3D_OK;
}

}  // extern "C"

// Stage orchestration: allocation of named device arrays, launch order, and the
// few host<->device handshakes (output sizes) each stage needs.
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "ctx.cuh"
#include "kernels.cuh"
#include "stages.cuh"

using msc3d_dev::Dims;

namespace msc3d_stage {

#define TRY(x)                              \
    do {                                    \
        const int _rc = (x);                \
        if (_rc != MSC3D_OK) return _rc;    \
    } while (0)

int gradient(msc3d_ctx* ctx, bool with_forests) {
    const Dims& d = ctx->dims;
    auto* codes = static_cast<std::uint8_t*>(ctx->ensure("codes", d.n_cells, 1));
    if (!codes) return MSC3D_ERR_NOMEM;
    std::uint32_t* p0 = nullptr;
    std::uint32_t* p3 = nullptr;
    if (with_forests) {
        p0 = static_cast<std::uint32_t*>(ctx->ensure("parent0", d.n_verts, 4));
        p3 = static_cast<std::uint32_t*>(ctx->ensure("parent3", d.n_cubes, 4));
        if (!p0 || !p3) return MSC3D_ERR_NOMEM;
    }
    return msc3d_dev::launch_gradient(ctx->values, ctx->value_type, d, codes, p0, p3, ctx->stream);
}

int critical(msc3d_ctx* ctx) {
    const Dims& d = ctx->dims;
    const auto* codes = ctx->ptr<std::uint8_t>("codes");
    TRY(msc3d_dev::launch_critical_count(codes, d, ctx->d_small, ctx->stream, ctx->num_sms));
    TRY(ctx->fetch_small(4));
    std::uint64_t n[4];
    std::memcpy(n, ctx->h_small, sizeof n);
    const int w = ctx->id_width();
    void* outs[4];
    for (int k = 0; k < 4; ++k) {
        outs[k] = ctx->ensure("crit" + std::to_string(k), n[k], w);
        if (!outs[k]) return MSC3D_ERR_NOMEM;
        ctx->scalars["c" + std::to_string(k)] = static_cast<std::int64_t>(n[k]);
    }
    TRY(msc3d_dev::launch_critical_compact(codes, d, ctx->ws, outs, w, ctx->d_small + 8,
                                           ctx->stream));
    ctx->scalars["euler"] = static_cast<std::int64_t>(n[0]) - static_cast<std::int64_t>(n[1]) +
                            static_cast<std::int64_t>(n[2]) - static_cast<std::int64_t>(n[3]);
    return MSC3D_OK;
}

int forest(msc3d_ctx* ctx, int dim) {
    const Dims& d = ctx->dims;
    const std::uint64_t n = dim == 0 ? d.n_verts : d.n_cubes;
    auto* p = static_cast<std::uint32_t*>(ctx->ensure(dim == 0 ? "parent0" : "parent3", n, 4));
    if (!p) return MSC3D_ERR_NOMEM;
    return msc3d_dev::launch_forest(ctx->ptr<std::uint8_t>("codes"), d, dim, p, ctx->stream,
                                    ctx->num_sms);
}

// find_roots with the reference's synchronous doubling: identical labels and the
// identical `rounds` count (extrema.cpp:79-101).
int roots_sync(msc3d_ctx* ctx, int dim) {
    const std::string pn = dim == 0 ? "parent0" : "parent3";
    const std::string ln = dim == 0 ? "label0" : "label3";
    const std::uint64_t n = ctx->count(pn);
    auto* a = static_cast<std::uint32_t*>(ctx->ensure(ln, n, 4));
    auto* b = static_cast<std::uint32_t*>(ctx->ensure(ln + ".tmp", n, 4));
    if (!a || !b) return MSC3D_ERR_NOMEM;
    if (n) MSC3D_CUDA_TRY(cudaMemcpyAsync(a, ctx->ptr<void>(pn), n * 4, cudaMemcpyDeviceToDevice, ctx->stream));
    int rounds = 0;
    auto* changed = reinterpret_cast<unsigned int*>(ctx->d_small);
    while (n) {
        MSC3D_CUDA_TRY(cudaMemsetAsync(changed, 0, 4, ctx->stream));
        TRY(msc3d_dev::launch_double_round(a, b, n, changed, ctx->stream, ctx->num_sms));
        TRY(ctx->fetch_small(1));
        if ((ctx->h_small[0] & 0xffffffffu) == 0) break;
        ++rounds;
        std::swap(a, b);
    }
    // make sure the named array holds the final labels
    if (n && a != ctx->ptr<std::uint32_t>(ln))
        MSC3D_CUDA_TRY(cudaMemcpyAsync(ctx->ptr<void>(ln), a, n * 4, cudaMemcpyDeviceToDevice, ctx->stream));
    ctx->scalars[dim == 0 ? "rounds0" : "rounds3"] = rounds;
    return MSC3D_OK;
}

// Roots for the pipeline: in-place jumping on the parent array itself (it becomes
// the label array).  Checks convergence every round.
int roots_fast(msc3d_ctx* ctx, int dim) {
    const std::string pn = dim == 0 ? "parent0" : "parent3";
    const std::uint64_t n = ctx->count(pn);
    auto* p = ctx->ptr<std::uint32_t>(pn);
    auto* changed = reinterpret_cast<unsigned int*>(ctx->d_small + 16 + dim);
    int rounds = 0;
    while (n) {
        MSC3D_CUDA_TRY(cudaMemsetAsync(changed, 0, 4, ctx->stream));
        TRY(msc3d_dev::launch_jump_round(p, n, changed, ctx->stream, ctx->num_sms));
        unsigned int h = 0;
        MSC3D_CUDA_TRY(cudaMemcpyAsync(&ctx->h_small[16 + dim], changed, 4, cudaMemcpyDeviceToHost, ctx->stream));
        MSC3D_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
        h = static_cast<unsigned int>(ctx->h_small[16 + dim] & 0xffffffffu);
        ++rounds;
        if (!h) break;
        if (rounds > 64) return MSC3D_ERR_RUNTIME;
    }
    ctx->scalars[dim == 0 ? "jump_rounds0" : "jump_rounds3"] = rounds;
    return MSC3D_OK;
}

int se_arcs(msc3d_ctx* ctx) {
    const Dims& d = ctx->dims;
    const auto* codes = ctx->ptr<std::uint8_t>("codes");
    const int w = ctx->id_width();
    TRY(msc3d_dev::launch_saddle_count(codes, d, ctx->d_small, ctx->stream, ctx->num_sms));
    TRY(ctx->fetch_small(1));
    const std::uint64_t ns = ctx->h_small[0];
    void* sad = ctx->ensure("se_saddles_all", ns, w);
    auto* slot = static_cast<std::uint64_t*>(ctx->ensure("se_slot", 2 * ns, 8));
    auto* cnt = static_cast<std::uint32_t*>(ctx->ensure("se_cnt", ns, 4));
    auto* off = static_cast<std::uint64_t*>(ctx->ensure("se_off", ns, 8));
    if (!sad || !slot || !cnt || !off) return MSC3D_ERR_NOMEM;
    TRY(msc3d_dev::launch_saddle_compact(codes, d, ctx->ws, sad, w, ctx->d_small + 8, ctx->stream));
    TRY(msc3d_dev::launch_se_slots(codes, d, sad, ns, w, ctx->ptr<std::uint32_t>("label0"),
                                   ctx->ptr<std::uint32_t>("label3"), slot, cnt, ctx->stream,
                                   ctx->num_sms));
    TRY(msc3d_dev::scan_u32(cnt, ns, off, ctx->d_small, ctx->ws, ctx->stream));
    TRY(ctx->fetch_small(1));
    const std::uint64_t na = ns ? ctx->h_small[0] : 0;
    void* os = ctx->ensure("se_saddle", na, w);
    void* oe = ctx->ensure("se_extremum", na, w);
    auto* om = static_cast<std::uint32_t*>(ctx->ensure("se_mult", na, 4));
    if (!os || !oe || !om) return MSC3D_ERR_NOMEM;
    return msc3d_dev::launch_se_write(sad, ns, w, slot, off, os, oe, om, ctx->stream, ctx->num_sms);
}

int mark(msc3d_ctx*, const void*, std::uint64_t) { return MSC3D_ERR_STATE; }
int minor(msc3d_ctx*) { return MSC3D_ERR_STATE; }
int count(msc3d_ctx*) { return MSC3D_ERR_STATE; }
int count_minor(msc3d_ctx*, const void*, std::uint64_t, const void*, std::uint64_t, const void*,
                std::uint64_t, const std::uint32_t* const*, const std::uint32_t* const*,
                const std::uint64_t* const*, const std::uint64_t*, int) {
    return MSC3D_ERR_STATE;
}
int compute(msc3d_ctx*, int, double*) { return MSC3D_ERR_STATE; }

}  // namespace msc3d_stage

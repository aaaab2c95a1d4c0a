// Stage orchestration: allocation of named device arrays, launch order, and the
// few host<->device handshakes (output sizes) each stage needs.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"
#include "ctx.cuh"
#include "host_decode.hpp"
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
    // per-dimension critical counts come for free from the gradient kernel; stars
    // with tied values are finished by the deferred slow-path kernel
    std::uint32_t* lists[3] = {static_cast<std::uint32_t*>(ctx->ensure("star_list16", 2 * d.n_verts, 4)),
                               static_cast<std::uint32_t*>(ctx->ensure("star_list32", 2 * d.n_verts, 4)),
                               static_cast<std::uint32_t*>(ctx->ensure("star_list_ties", d.n_verts, 4))};
    if (!lists[0] || !lists[1] || !lists[2]) return MSC3D_ERR_NOMEM;
    ctx->crit_counts_valid = true;
    return msc3d_dev::launch_gradient(ctx->values, ctx->value_type, d, codes, p0, p3, ctx->stream,
                                      reinterpret_cast<unsigned long long*>(ctx->d_small + 40), lists,
                                      reinterpret_cast<unsigned long long*>(ctx->d_small + 44),
                                      ctx->num_sms);
}

int critical(msc3d_ctx* ctx) {
    const Dims& d = ctx->dims;
    const auto* codes = ctx->ptr<std::uint8_t>("codes");
    std::uint64_t n[4];
    if (ctx->crit_counts_valid) {
        TRY(ctx->fetch_small(44));
        std::memcpy(n, ctx->h_small + 40, sizeof n);
    } else {
        TRY(msc3d_dev::launch_critical_count(codes, d, ctx->d_small, ctx->stream, ctx->num_sms));
        TRY(ctx->fetch_small(4));
        std::memcpy(n, ctx->h_small, sizeof n);
    }
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

// ---------------------------------------------------------------------------------
// mark_reachable (saddle_graph.cpp:26-86)
// ---------------------------------------------------------------------------------
namespace {

template <typename T>
std::vector<T> sorted_unique(const T* p, std::uint64_t n) {
    std::vector<T> v(p, p + n);
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
    return v;
}

// Successor table of the current codes (dag.cu): 2 bytes per dense edge.
int succ_table(msc3d_ctx* ctx) {
    const Dims& d = ctx->dims;
    // (+32: junction_bits reads whole 32-word groups)
    auto* succ = static_cast<std::uint16_t*>(ctx->ensure("succ", 3 * d.n_verts + 32, 2));
    if (!succ) return MSC3D_ERR_NOMEM;
    return msc3d_dev::launch_succ_table(ctx->ptr<std::uint8_t>("codes"), d, succ, ctx->stream, ctx->num_sms);
}

int bfs(msc3d_ctx* ctx, const void* d_sources, std::uint64_t n_src) {
    const Dims& d = ctx->dims;
    const auto* codes = ctx->ptr<std::uint8_t>("codes");
    const int w = ctx->id_width();
    const std::uint64_t nde = 3 * d.n_verts;
    const std::uint64_t nwords = (nde + 31) / 32;
    // dense edge ids de = 3*vertex + axis and frontier entries are u32
    if (nde >= 0xffffffffull) return MSC3D_ERR_INVALID;
    TRY(succ_table(ctx));
    auto* bitmap = static_cast<unsigned int*>(ctx->ensure("visited", nwords, 4));
    if (!bitmap) return MSC3D_ERR_NOMEM;
    // [0] rounds (~0: a level overflowed the frontier buffers) [1] claims
    // [2 + r] device time at the start of round r (ns)
    auto* stats = static_cast<unsigned long long*>(ctx->ensure("reach_stats", 2 + 256, 8));
    if (!stats) return MSC3D_ERR_NOMEM;
    auto* cnt = reinterpret_cast<unsigned long long*>(ctx->d_small + 48);     // 3 counters
    auto* bad = reinterpret_cast<unsigned int*>(ctx->d_small + 51);
    // Frontier buffers: a level has at most 4x the nodes of the one before (<= 4
    // successors per 1-cell) and the measured levels stay near the source count, so
    // they start at 4 x sources (not 3V entries each: 2 x 12.9 GB at 2^30 vertices);
    // a level that does not fit is detected in the kernel and the BFS reruns with
    // buffers of every dense edge.
    std::uint64_t fcap = std::min<std::uint64_t>(nde, std::max<std::uint64_t>(4 * n_src, 1ull << 22));
    if (ctx->frontier_cap) fcap = std::min<std::uint64_t>(nde, std::max<std::uint64_t>(ctx->frontier_cap, n_src));
    for (int attempt = 0;; ++attempt) {
        auto* fa = static_cast<std::uint32_t*>(ctx->ensure("frontier_a", fcap, 4));
        auto* fb = static_cast<std::uint32_t*>(ctx->ensure("frontier_b", fcap, 4));
        if (!fa || !fb) return MSC3D_ERR_NOMEM;
        MSC3D_CUDA_TRY(cudaMemsetAsync(bitmap, 0, nwords * 4, ctx->stream));
        MSC3D_CUDA_TRY(cudaMemsetAsync(stats, 0, 2 * 8, ctx->stream));
        ctx->h_small[48] = n_src;
        for (int k = 49; k < 54; ++k) ctx->h_small[k] = 0;
        MSC3D_CUDA_TRY(cudaMemcpyAsync(cnt, &ctx->h_small[48], 6 * 8, cudaMemcpyHostToDevice, ctx->stream));
        // seeds: validated 1-saddles, their bits set (saddle_graph.cpp:29-41)
        TRY(msc3d_dev::launch_bfs_sources(codes, d, d_sources, n_src, w, bitmap, fa, bad, ctx->stream,
                                          ctx->num_sms));
        if (n_src)
            TRY(msc3d_dev::launch_reach(ctx->ptr<std::uint16_t>("succ"), d, bitmap, fa, fb, fcap, cnt, stats,
                                        ctx->stream, ctx->num_sms));
        MSC3D_CUDA_TRY(cudaMemcpyAsync(ctx->d_small + 52, stats, 2 * 8, cudaMemcpyDeviceToDevice, ctx->stream));
        TRY(ctx->fetch_small(54));
        if (ctx->h_small[51] & 0xffffffffu) return MSC3D_ERR_INVALID;  // saddle_graph.cpp:29-31
        if (ctx->h_small[52] != ~0ull) break;
        if (fcap >= nde) return MSC3D_ERR_RUNTIME;  // (cannot happen: a level holds distinct edges)
        ctx->scalars["bfs_frontier_retries"] = attempt + 1;
        fcap = nde;
    }
    ctx->scalars["bfs_frontier_cap"] = static_cast<std::int64_t>(fcap);
    const std::int64_t rounds = static_cast<std::int64_t>(ctx->h_small[52]);
    ctx->h_small[49] = ctx->h_small[53];
    ctx->scalars["bfs_levels"] = rounds;  // BFS levels
    ctx->scalars["dag_nodes"] = static_cast<std::int64_t>(n_src + ctx->h_small[49]);
    ctx->scalars["dag_sources"] = static_cast<std::int64_t>(n_src);
    return MSC3D_OK;
}

int marked_lists(msc3d_ctx* ctx) {
    const Dims& d = ctx->dims;
    const auto* codes = ctx->ptr<std::uint8_t>("codes");
    const int w = ctx->id_width();
    auto* marked = static_cast<std::uint8_t*>(ctx->ensure("marked", d.n_cells, 1));
    if (!marked) return MSC3D_ERR_NOMEM;
    MSC3D_CUDA_TRY(cudaMemsetAsync(marked, 0, d.n_cells, ctx->stream));
    const std::uint64_t nwords = ctx->count("visited");
    TRY(msc3d_dev::launch_marked_bytes(codes, d, ctx->ptr<unsigned int>("visited"), nwords, marked,
                                       ctx->stream, ctx->num_sms));
    TRY(msc3d_dev::launch_marked_critical_count(codes, marked, d, ctx->d_small, ctx->stream, ctx->num_sms));
    TRY(ctx->fetch_small(4));
    const std::uint64_t n1 = ctx->h_small[1], n2 = ctx->h_small[2];
    void* outs[4] = {nullptr, ctx->ensure("one_saddles", n1, w), ctx->ensure("two_saddles", n2, w),
                     nullptr};
    if (!outs[1] || !outs[2]) return MSC3D_ERR_NOMEM;
    return msc3d_dev::launch_marked_critical_compact(codes, marked, d, ctx->ws, outs, w,
                                                     ctx->d_small + 8, ctx->stream);
}

}  // namespace

int mark(msc3d_ctx* ctx, const void* host_sources, std::uint64_t n_sources) {
    const int w = ctx->id_width();
    std::uint64_t n = 0;
    if (!host_sources) {
        TRY(critical(ctx));  // the codes may have changed since the last extraction
        n = ctx->count("crit1");
        void* p = ctx->ensure("sources", n, w);
        if (!p) return MSC3D_ERR_NOMEM;
        if (n) MSC3D_CUDA_TRY(cudaMemcpyAsync(p, ctx->ptr<void>("crit1"), n * w, cudaMemcpyDeviceToDevice, ctx->stream));
    } else {
        // The reference skips duplicate sources (saddle_graph.cpp:37-41); sources are
        // kept in ascending order, which is also the order of one_saddles.
        if (w == 4) {
            auto v = sorted_unique(static_cast<const std::uint32_t*>(host_sources), n_sources);
            n = v.size();
            void* p = ctx->ensure("sources", n, 4);
            if (!p) return MSC3D_ERR_NOMEM;
            if (n) MSC3D_CUDA_TRY(cudaMemcpyAsync(p, v.data(), n * 4, cudaMemcpyHostToDevice, ctx->stream));
            MSC3D_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
        } else {
            auto v = sorted_unique(static_cast<const std::uint64_t*>(host_sources), n_sources);
            n = v.size();
            void* p = ctx->ensure("sources", n, 8);
            if (!p) return MSC3D_ERR_NOMEM;
            if (n) MSC3D_CUDA_TRY(cudaMemcpyAsync(p, v.data(), n * 8, cudaMemcpyHostToDevice, ctx->stream));
            MSC3D_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
        }
    }
    TRY(bfs(ctx, ctx->ptr<void>("sources"), n));
    return marked_lists(ctx);
}

// ---------------------------------------------------------------------------------
// path counting over the device DAG
// ---------------------------------------------------------------------------------
namespace {

// src_ids[0, n1): the BFS sources (ascending 1-saddle ids, already traversed by bfs());
// term_list: ascending 2-saddle ids whose positions key the count vectors.  Output
// ranks into those lists.
// `place` (optional) receives the output length and returns where to write the
// (one, two, paths) triples and the bases added to the ranks; default: the arrays
// "ss_one_rank", "ss_two_rank", "ss_paths" with ranks as they are.
struct CountOut {
    std::uint32_t* one = nullptr;
    std::uint32_t* two = nullptr;
    std::uint64_t* paths = nullptr;
    std::uint32_t base_one = 0, base_two = 0;
};
// The exact A* decision behind a "maybe" of the dead-junction bound (dag.cu, JRec):
// the minor of this BFS (saddle_graph.cpp:121-217) built on the device and
// count_paths' own overflow rule applied to it (count_minor: forward saturating
// totals, then the exact per-source check).  Only runs when some source's paths into
// dead junctions may reach 2^64; it clobbers the minor/count_minor scratch arrays.
int exact_dead_overflow(msc3d_ctx* ctx) {
    TRY(marked_lists(ctx));
    TRY(minor(ctx));
    const int w = ctx->id_width();
    static const char* kLists[4] = {"s1_to_j", "j_to_j", "j_to_s2", "s1_to_s2"};
    std::vector<std::uint32_t> src[4], dst[4];
    std::vector<std::uint64_t> mult[4];
    const std::uint32_t* ps[4];
    const std::uint32_t* pd[4];
    const std::uint64_t* pm[4];
    std::uint64_t cnt[4];
    for (int k = 0; k < 4; ++k) {
        const std::string n = kLists[k];
        cnt[k] = ctx->count(n + ".src");
        src[k].resize(cnt[k]);
        dst[k].resize(cnt[k]);
        mult[k].resize(cnt[k]);
        if (cnt[k]) {
            MSC3D_CUDA_TRY(cudaMemcpy(src[k].data(), ctx->ptr<void>(n + ".src"), cnt[k] * 4, cudaMemcpyDeviceToHost));
            MSC3D_CUDA_TRY(cudaMemcpy(dst[k].data(), ctx->ptr<void>(n + ".dst"), cnt[k] * 4, cudaMemcpyDeviceToHost));
            MSC3D_CUDA_TRY(cudaMemcpy(mult[k].data(), ctx->ptr<void>(n + ".mult"), cnt[k] * 8, cudaMemcpyDeviceToHost));
        }
        ps[k] = src[k].data();
        pd[k] = dst[k].data();
        pm[k] = mult[k].data();
    }
    return count_minor(ctx, nullptr, ctx->count("one_saddles"), nullptr, ctx->count("junctions"), nullptr,
                       ctx->count("two_saddles"), ps, pd, pm, cnt, w);
}

int dag_count(msc3d_ctx* ctx, const void* src_ids, std::uint64_t n1, const std::string& term_list,
              const std::function<int(std::uint64_t, CountOut*)>& place = nullptr) {
    const Dims& d = ctx->dims;
    const int w = ctx->id_width();
    const cudaStream_t s = ctx->stream;
    const int sms = ctx->num_sms;
    const std::uint64_t nde = 3 * d.n_verts;
    const std::uint64_t nwords = (nde + 31) / 32;
    const auto* bitmap = ctx->ptr<unsigned int>("visited");
    const auto* succ = ctx->ptr<std::uint16_t>("succ");
    auto* flags = reinterpret_cast<unsigned int*>(ctx->d_small + 26);  // [0] overflow [1] pool [2] cycle
    MSC3D_CUDA_TRY(cudaMemsetAsync(flags, 0, 16, s));

    // junctions: bitmap + per-word ranks + list in dense-edge order
    // 2-saddle ranks for the walks' terminal lookups: a u32 per dense quad (one load)
    // up to 2^28 vertices (3 GB), above that rank words in cell order (N/4 bytes)
    const bool use_tmap = d.n_verts <= (1ull << 28) && !ctx->term_rank_words;
    std::uint32_t* tmap = nullptr;
    void* trank = nullptr;
    if (use_tmap) {
        ctx->release("term_rank");
        tmap = static_cast<std::uint32_t*>(ctx->ensure("tmap", nde, 4));
        if (!tmap) return MSC3D_ERR_NOMEM;
        TRY(msc3d_dev::launch_scatter_quad_rank(ctx->ptr<void>(term_list), ctx->count(term_list), w, d, tmap, s, sms));
    } else {
        ctx->release("tmap");
        trank = ctx->ensure("term_rank", d.n_cells / 32 + 1, 8);
        if (!trank) return MSC3D_ERR_NOMEM;
        TRY(msc3d_dev::launch_term_rank(ctx->ptr<void>(term_list), ctx->count(term_list), w, d.n_cells, trank, s,
                                        sms));
    }
    auto* jbits = static_cast<unsigned int*>(ctx->ensure("jbits", nwords, 4));
    auto* jcnt = static_cast<std::uint32_t*>(ctx->ensure("jcount", nwords, 4));
    auto* woff = static_cast<std::uint64_t*>(ctx->ensure("joff", nwords, 8));
    if (!jbits || !jcnt || !woff) return MSC3D_ERR_NOMEM;
    MSC3D_CUDA_TRY(cudaMemsetAsync(ctx->d_small + 50, 0, 8, s));
    TRY(msc3d_dev::launch_junction_bits(succ, bitmap, nwords, jbits, jcnt,
                                        reinterpret_cast<unsigned long long*>(ctx->d_small + 50), s, sms));
    TRY(msc3d_dev::scan_u32(jcnt, nwords, woff, ctx->d_small, ctx->ws, s));
    TRY(ctx->fetch_small(1));
    const std::uint64_t nj = ctx->h_small[0];
    const std::uint64_t nn = nj + n1;
    // branch destinations are u32 ranks with kTerm (bit 31) marking 2-saddles
    if (nj >= 0x80000000ull || ctx->count(term_list) >= 0x80000000ull) return MSC3D_ERR_INVALID;
    ctx->scalars["junctions"] = static_cast<std::int64_t>(nj);
    auto* jlist = static_cast<std::uint32_t*>(ctx->ensure("jlist", nj, 4));
    void* node = ctx->ensure("jnode", nn, msc3d_dev::node_rec_bytes());
    auto* jdest = static_cast<char*>(ctx->ensure("jdest", std::max<std::uint64_t>(nn, 1), 16));  // branch destinations
    auto* pending = static_cast<std::uint8_t*>(ctx->ensure("pending", nn + 4, 1));  // (+4: word-wide atomics)
    auto* pending0 = static_cast<std::uint8_t*>(ctx->ensure("pending0", nn + 4, 1));
    auto* indeg = static_cast<std::uint32_t*>(ctx->ensure("indeg", nj, 4));
    auto* fwd = static_cast<std::uint32_t*>(ctx->ensure("jfwd", nj, 4));
    auto* ovoff = static_cast<std::uint64_t*>(ctx->ensure("ovoff", nj, 8));
    void* rec = ctx->ensure("jrec", nj, msc3d_dev::count_rec_bytes());
    auto* slen = static_cast<std::uint32_t*>(ctx->ensure("slen", n1, 4));
    auto* soff = static_cast<std::uint64_t*>(ctx->ensure("soff", n1, 8));
    auto* ptop = static_cast<unsigned long long*>(ctx->ensure("pool_top", msc3d_dev::count_arenas(), 8));
    // Kahn's frontiers hold junctions; the BFS buffers are reused (grown if needed)
    const std::uint64_t fcap = std::max<std::uint64_t>(std::max<std::uint64_t>(ctx->count("frontier_a"), nn), 1024);
    auto* fa = static_cast<std::uint32_t*>(ctx->ensure("frontier_a", fcap, 4));
    auto* fb = static_cast<std::uint32_t*>(ctx->ensure("frontier_b", fcap, 4));
    if (!jlist || !node || !jdest || !pending || !pending0 || !indeg || !fwd || !ovoff || !rec ||
        !slen || !soff || !ptop || !fa || !fb)
        return MSC3D_ERR_NOMEM;
    void* jrank = ctx->ensure("jrank", nwords, 8);
    if (!jrank) return MSC3D_ERR_NOMEM;
    TRY(msc3d_dev::launch_junction_list(jbits, nwords, woff, jrank, jlist, s, sms));

    // branch walks (saddle_graph.cpp:139-202): destinations and pending children
    auto* predone = static_cast<unsigned int*>(ctx->ensure("predone", (nj + 31) / 32 + 1, 4));
    if (!predone) return MSC3D_ERR_NOMEM;
    auto* n_predone = reinterpret_cast<unsigned long long*>(ctx->d_small + 30);
    MSC3D_CUDA_TRY(cudaMemsetAsync(n_predone, 0, 8, s));
    // (the junction walks also flag the pass-through junctions: fwd, ptbits)
    auto* ptbits = static_cast<unsigned int*>(ctx->ensure("ptbits", (nj + 31) / 32 + 1, 4));
    if (!ptbits) return MSC3D_ERR_NOMEM;
    TRY(msc3d_dev::launch_walk(succ, d, jrank, tmap, trank, jlist, nullptr, w, nj, jdest, pending, flags, rec, nullptr,
                               predone, n_predone, fwd, ptbits, s, sms));
    TRY(msc3d_dev::launch_walk(succ, d, jrank, tmap, trank, nullptr, src_ids, w, n1,
                               jdest + nj * 16, pending + nj, flags, nullptr, slen, nullptr, nullptr, nullptr, nullptr, s,
                               sms));
    // pass-through junctions (one live branch, to a junction: P(j) = P(child)) are
    // contracted away by pointer jumping

    {  // pointer jumping to the end of pass-through chains, all rounds in one launch
        auto* jflags = reinterpret_cast<unsigned int*>(ctx->d_small + 23);
        auto* jrounds = reinterpret_cast<unsigned long long*>(ctx->d_small + 25);
        MSC3D_CUDA_TRY(cudaMemsetAsync(ctx->d_small + 23, 0, 24, s));
        auto* conv = static_cast<unsigned int*>(ctx->ensure("jump_conv_pt", nj / 32 + 1, 4));
        if (!conv) return MSC3D_ERR_NOMEM;
        TRY(msc3d_dev::launch_jump_all(fwd, nj, nullptr, 0, conv, jflags, jrounds, s, sms));
    }
    if (nj) MSC3D_CUDA_TRY(cudaMemsetAsync(indeg, 0, nj * 4, s));
    auto* n_skip = reinterpret_cast<unsigned long long*>(ctx->d_small + 19);
    auto* ovq_n = reinterpret_cast<unsigned long long*>(ctx->d_small + 20);
    MSC3D_CUDA_TRY(cudaMemsetAsync(ctx->d_small + 19, 0, 16, s));
    // overflow queue (parents beyond the inline ones): reuse a frontier buffer
    // (>= nn u32: room for nn/4 entries >> the measured ~0.1% of nodes)
    void* ovq = fa;
    const std::uint64_t ovq_cap = fcap / 4;
    auto* ready = static_cast<std::uint32_t*>(ctx->ensure("ready0", std::max<std::uint64_t>(nj, 1), 4));
    if (!ready) return MSC3D_ERR_NOMEM;
    auto* n_ready = reinterpret_cast<unsigned long long*>(ctx->d_small + 77);
    MSC3D_CUDA_TRY(cudaMemsetAsync(n_ready, 0, 8, s));
    TRY(msc3d_dev::launch_rewrite(node, jdest, nj, nn, fwd, ptbits, predone, pending, indeg, ovq, ovq_n, ovq_cap, n_skip,
                                  ready, n_ready, s, sms));
    // parents beyond the inline ones: an overflow list
    TRY(msc3d_dev::launch_parent_overflow(indeg, nj, ovoff, reinterpret_cast<unsigned long long*>(ctx->d_small), s,
                                          sms));
    TRY(ctx->fetch_small(28));
    if (static_cast<unsigned int>(ctx->h_small[27])) return MSC3D_ERR_RUNTIME;  // cycle in a walk
    if (nj && ctx->h_small[25] > 64) return MSC3D_ERR_RUNTIME;                  // cycle of pass-through junctions
    const std::uint64_t nov = nj ? ctx->h_small[0] : 0;
    const std::uint64_t nskip = ctx->h_small[19];
    const std::uint64_t nq = ctx->h_small[20];
    if (nq > ovq_cap) return MSC3D_ERR_NOMEM;  // parent overflow queue capacity, not a cycle
    if (nq != nov) return MSC3D_ERR_RUNTIME;
    ctx->scalars["junctions_contracted"] = static_cast<std::int64_t>(nskip);
    auto* rsrc = static_cast<std::uint32_t*>(ctx->ensure("rsrc", std::max<std::uint64_t>(nov, 1), 4));
    if (!rsrc) return MSC3D_ERR_NOMEM;
    TRY(msc3d_dev::launch_fill_parents(node, nj, indeg, ovoff, ovq, nq, rsrc, s, sms));
    if (nn) MSC3D_CUDA_TRY(cudaMemcpyAsync(pending0, pending, nn, cudaMemcpyDeviceToDevice, s));

    // count vectors, "last child continues"; grow the pool and rerun if it ran out
    const std::uint64_t m = static_cast<std::uint64_t>(ctx->scalars["dag_nodes"]);
    const std::uint64_t arenas = static_cast<std::uint64_t>(msc3d_dev::count_arenas());
    // pool space is reserved per junction by its input length (rounded up to 4)
    std::uint64_t pcap = std::max<std::uint64_t>(arenas << 16, m + m / 2);
    auto* kcnt = reinterpret_cast<unsigned long long*>(ctx->d_small + 55);  // 3 counters
    // [0] rounds [1 + r] device time at the start of round r (ns)
    auto* kstats = static_cast<unsigned long long*>(ctx->ensure("count_stats", 1 + 256, 8));
    if (!kstats) return MSC3D_ERR_NOMEM;
    auto* done = reinterpret_cast<unsigned long long*>(ctx->d_small + 59);
    msc3d_dev::CountLaunch L{};
    for (int attempt = 0;; ++attempt) {
        L.pool_key = static_cast<std::uint32_t*>(ctx->ensure("pool_key", pcap, 4));
        L.pool_cnt = static_cast<std::uint64_t*>(ctx->ensure("pool_cnt", pcap, 8));
        if (!L.pool_key || !L.pool_cnt) return MSC3D_ERR_NOMEM;
        L.node = node;
        L.dest = jdest;
        L.pending = pending;
        L.pending0 = pending0;
        L.rsrc = rsrc;
        L.rec = rec;
        L.pool_top = ptop;
        L.arena_cap = (pcap / arenas) & ~3ull;
        L.slen = slen;
        L.nj = nj;
        L.n1 = n1;
        L.fa = fa;
        L.fb = fb;
        L.cnt = kcnt;
        L.stats = kstats;
        L.done = done;
        L.flags = flags;
        L.diag = nullptr;
        L.heavy_q = static_cast<std::uint32_t*>(ctx->ensure("heavy_q", std::max<std::uint64_t>(nn, 1), 4));
        L.heavy_n = reinterpret_cast<unsigned long long*>(ctx->d_small + 61);
        L.resume = reinterpret_cast<unsigned long long*>(ctx->d_small + 64);  // 3 words
        L.heavy_rounds = reinterpret_cast<unsigned long long*>(ctx->d_small + 70);  // 6 words
        L.indeg = indeg;
        L.ovoff = ovoff;
        L.switch_below = ctx->kahn_switch_below;
        L.async_tail = ctx->kahn_async;
        L.qctl = static_cast<unsigned long long*>(ctx->ensure("kahn_qctl", 64, 8));
        if (!L.qctl) return MSC3D_ERR_NOMEM;
        L.n_skip = n_skip;
        L.n_predone = n_predone;
        L.ready = ready;
        L.n_ready = n_ready;
        if (!L.heavy_q) return MSC3D_ERR_NOMEM;
        MSC3D_CUDA_TRY(cudaMemsetAsync(ctx->d_small + 61, 0, 16, s));
        MSC3D_CUDA_TRY(cudaMemsetAsync(ctx->d_small + 70, 0, 48, s));
        if (std::getenv("MSC3D_DIAG")) {
            L.diag = static_cast<unsigned long long*>(ctx->ensure("count_diag", 1024, 8));
            if (L.diag) MSC3D_CUDA_TRY(cudaMemsetAsync(L.diag, 0, 1024 * 8, s));
        }
        MSC3D_CUDA_TRY(cudaMemsetAsync(flags, 0, 8, s));
        MSC3D_CUDA_TRY(cudaMemsetAsync(flags + 3, 0, 4, s));  // dead-junction "maybe"
        MSC3D_CUDA_TRY(cudaMemsetAsync(ptop, 0, arenas * 8, s));
        MSC3D_CUDA_TRY(cudaMemsetAsync(ctx->d_small + 55, 0, 5 * 8, s));
        if (nn) MSC3D_CUDA_TRY(cudaMemcpyAsync(pending, pending0, nn, cudaMemcpyDeviceToDevice, s));
        TRY(msc3d_dev::launch_count(L, s, sms));
        MSC3D_CUDA_TRY(cudaMemcpyAsync(ctx->d_small + 58, kstats, 8, cudaMemcpyDeviceToDevice, s));
        TRY(ctx->fetch_small(60));
        ctx->scalars["count_levels"] = static_cast<std::int64_t>(ctx->h_small[58]);
        const unsigned int pool_full = static_cast<unsigned int>(ctx->h_small[26] >> 32);
        if (pool_full) {
            if (attempt > 8) return MSC3D_ERR_NOMEM;
            pcap *= 2;
            continue;
        }
        // junctions finished by Kahn + by the walk (leaves) + contracted = all, else a cycle
        if (ctx->h_small[59] + ctx->h_small[30] != nj - nskip) return MSC3D_ERR_RUNTIME;  // path_matrix.cpp:202-203
        break;
    }
    {
        MSC3D_CUDA_TRY(cudaMemcpyAsync(ctx->d_small + 128, ptop, arenas * 8, cudaMemcpyDeviceToDevice, s));
        TRY(ctx->fetch_range(128, static_cast<int>(arenas)));
        std::uint64_t used = 0;
        for (std::uint64_t k = 0; k < arenas; ++k) used += ctx->h_small[128 + k];
        ctx->scalars["pool_entries"] = static_cast<std::int64_t>(used);
    }

    // 1-saddles: merged lengths (those the walk did not finish), offsets, sorted output
    TRY(msc3d_dev::launch_source_len(L, s, sms));
    TRY(msc3d_dev::scan_u32(slen, n1, soff, ctx->d_small, ctx->ws, s));
    TRY(ctx->fetch_small(28));
    if (ctx->h_small[26] & 0xffffffffu) return MSC3D_ERR_OVERFLOW;
    const std::uint64_t nout = n1 ? ctx->h_small[0] : 0;
    if (ctx->h_small[27] >> 32) {  // some source's paths into dead junctions may reach 2^64
        ctx->scalars["dead_overflow_checks"] += 1;
        TRY(exact_dead_overflow(ctx));
    }
    ctx->scalars["arcs_ss"] = static_cast<std::int64_t>(nout);
    CountOut o;
    if (place) {
        TRY(place(nout, &o));
    } else {
        o.one = static_cast<std::uint32_t*>(ctx->ensure("ss_one_rank", nout, 4));
        o.two = static_cast<std::uint32_t*>(ctx->ensure("ss_two_rank", nout, 4));
        o.paths = static_cast<std::uint64_t*>(ctx->ensure("ss_paths", nout, 8));
    }
    if (!o.one || !o.two || !o.paths) return MSC3D_ERR_NOMEM;
    TRY(msc3d_dev::launch_count_write(L, soff, o.one, o.two, o.paths, o.base_one, o.base_two, s, sms));
    TRY(ctx->fetch_small(27));
    if (ctx->h_small[26] & 0xffffffffu) return MSC3D_ERR_OVERFLOW;
    return MSC3D_OK;
}

}  // namespace

int count(msc3d_ctx* ctx) {
    TRY(dag_count(ctx, ctx->ptr<void>("sources"), ctx->count("sources"), "two_saddles"));
    const int w = ctx->id_width();
    const std::uint64_t n = static_cast<std::uint64_t>(ctx->scalars["arcs_ss"]);
    void* a = ctx->ensure("ss_one", n, w);
    void* b = ctx->ensure("ss_two", n, w);
    if (!a || !b) return MSC3D_ERR_NOMEM;
    TRY(msc3d_dev::launch_gather_ids(ctx->ptr<void>("sources"), ctx->ptr<std::uint32_t>("ss_one_rank"),
                                     n, w, a, ctx->stream, ctx->num_sms));
    return msc3d_dev::launch_gather_ids(ctx->ptr<void>("two_saddles"), ctx->ptr<std::uint32_t>("ss_two_rank"),
                                        n, w, b, ctx->stream, ctx->num_sms);
}

// ---------------------------------------------------------------------------------
// compute() (msc.cpp:57-147)
// ---------------------------------------------------------------------------------
namespace {

struct StageClock {
    cudaEvent_t ev[6] = {};
    bool ok = false;
    explicit StageClock(bool on) {
        if (!on) return;
        ok = true;
        for (auto& e : ev)
            if (cudaEventCreate(&e) != cudaSuccess) ok = false;
    }
    ~StageClock() {
        for (auto& e : ev)
            if (e) cudaEventDestroy(e);
    }
    void mark(int i, cudaStream_t s) {
        if (ok) cudaEventRecord(ev[i], s);
    }
};

}  // namespace

// Device-to-host copies of final outputs on a second stream, each enqueued as soon
// as its array is final, so they overlap the later stages.
struct Sink {
    msc3d_ctx* ctx;
    const msc3d_host_outputs* out;
    cudaStream_t cs = nullptr;
    std::vector<cudaEvent_t> evs;
    std::uint64_t bytes_moved = 0;  // D2H bytes of this delivery
    cudaStream_t producer = nullptr;  // stream that produced the arrays being copied (null: ctx->stream)
    cudaStream_t prod() const { return producer ? producer : ctx->stream; }
    std::chrono::steady_clock::time_point t_created = std::chrono::steady_clock::now();
    bool ok() const { return out != nullptr; }
    // development timeline (MSC3D_DIAG): [t0 on the compute stream, per copy: ready, start, end]
    bool diag = std::getenv("MSC3D_DIAG") != nullptr;
    std::vector<cudaEvent_t> tl;
    int copy(void* host, const void* dev, std::uint64_t bytes) {
        if (!out || !host || bytes == 0) return MSC3D_OK;
        if (!cs) {
            cs = ctx->copy_stream();
            if (!cs) return MSC3D_ERR_CUDA;
        }
        cudaEvent_t ev;
        MSC3D_CUDA_TRY(cudaEventCreateWithFlags(&ev, diag ? cudaEventDefault : cudaEventDisableTiming));
        evs.push_back(ev);
        MSC3D_CUDA_TRY(cudaEventRecord(ev, prod()));
        MSC3D_CUDA_TRY(cudaStreamWaitEvent(cs, ev, 0));
        cudaEvent_t a = nullptr, b = nullptr;
        if (diag) {
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            cudaEventRecord(a, cs);
            tl.push_back(ev);
            tl.push_back(a);
        }
        MSC3D_CUDA_TRY(cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, cs));
        bytes_moved += bytes;
        if (diag) {
            cudaEventRecord(b, cs);
            tl.push_back(b);
        }
        return MSC3D_OK;
    }
    // Narrow deliveries of the two arc arrays that compress: multiplicities (8 bytes
    // per arc, almost all < 255) as their byte, sources (sorted) as byte deltas with a
    // u32 head per chunk -- each with an (index, value) escape list (k_pack_mult /
    // k_pack_src).  The bytes go first on the copy stream, the escapes right behind
    // them (as many as the previous call of this block had, +25%, +64; the rest, if any, is
    // fetched later), and a host job per array decodes into the caller's buffer with
    // non-temporal stores, overlapping the block's remaining copies; finish() joins.
    // An escape list larger than its buffer falls back to copying the full array.
    struct Job {
        std::thread th;
        int rc = MSC3D_OK;
        std::uint64_t bytes = 0;  // D2H bytes the job moved itself
        std::string key;          // escape-count memo
        std::uint64_t n_esc = 0;
    };
    std::vector<std::unique_ptr<Job>> jobs;
    int copy_mult(std::uint64_t* host, const std::uint64_t* dev, std::uint64_t n, const char* tag) {
        if (!out || !host || n == 0) return MSC3D_OK;
        if (!ctx->d2h_narrow) return copy(host, dev, n * 8);
        return narrow(0, host, dev, n, std::string("mult_") + tag);
    }
    int copy_src(std::uint32_t* host, const std::uint32_t* dev, std::uint64_t n, const char* tag) {
        if (!out || !host || n == 0) return MSC3D_OK;
        if (!ctx->d2h_narrow) return copy(host, dev, n * 4);
        return narrow(1, host, dev, n, std::string("src_") + tag);
    }
    // kind 0: u64 multiplicities -> widen; kind 1: sorted u32 -> prefix-decode per chunk
    int narrow(int kind, void* host, const void* dev, std::uint64_t n, const std::string& t) {
        const std::uint64_t cap = ctx->d2h_escape_cap ? ctx->d2h_escape_cap : n / 16 + 1024;
        const std::uint64_t chunk = msc3d_dev::src_chunk();
        const std::uint64_t nh = kind == 1 ? (n + chunk - 1) / chunk : 0;
        auto* d8 = static_cast<std::uint8_t*>(ctx->ensure("d2h_b8_" + t, n, 1));
        auto* desc = static_cast<ulonglong2*>(ctx->ensure("d2h_esc_" + t, cap, 16));
        auto* dcnt = static_cast<unsigned long long*>(ctx->ensure("d2h_nesc_" + t, 1, 8));
        auto* dheads = static_cast<std::uint32_t*>(ctx->ensure("d2h_heads_" + t, nh + 1, 4));
        auto* h8 = static_cast<std::uint8_t*>(ctx->host_buf("b8_" + t, n));
        auto* hcnt = static_cast<unsigned long long*>(ctx->host_buf("nesc_" + t, 8));
        auto* hesc = static_cast<ulonglong2*>(ctx->host_buf("esc_" + t, cap * 16));
        auto* hheads = static_cast<std::uint32_t*>(ctx->host_buf("heads_" + t, (nh + 1) * 4));
        if (!d8 || !desc || !dcnt || !dheads || !h8 || !hcnt || !hesc || !hheads) return MSC3D_ERR_NOMEM;
        if (kind == 0)
            TRY(msc3d_dev::launch_pack_mult(static_cast<const std::uint64_t*>(dev), n, ctx->d2h_narrow_max, d8, desc,
                                            cap, dcnt, prod(), ctx->num_sms));
        else
            TRY(msc3d_dev::launch_pack_src(static_cast<const std::uint32_t*>(dev), n, ctx->d2h_narrow_max, d8, dheads,
                                           desc, cap, dcnt, prod(), ctx->num_sms));
        const std::uint64_t guess = std::min<std::uint64_t>(cap, ctx->d2h_esc_memo[t] * 5 / 4 + 64);
        TRY(copy(hcnt, dcnt, 8));
        TRY(copy(h8, d8, n));
        if (nh) TRY(copy(hheads, dheads, nh * 4));
        TRY(copy(hesc, desc, guess * 16));
        cudaEvent_t done;
        MSC3D_CUDA_TRY(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
        evs.push_back(done);
        MSC3D_CUDA_TRY(cudaEventRecord(done, cs));
        auto job = std::make_unique<Job>();
        Job* jp = job.get();
        jp->key = t;
        const int device = ctx->device;
        const bool dg = diag;
        const auto t_sink = t_created;
        jp->th = std::thread([=]() {
            auto ms_since = [&]() {
                return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_sink).count();
            };
            auto fail = [&](int rc) { jp->rc = rc; };
            if (cudaSetDevice(device) != cudaSuccess || cudaEventSynchronize(done) != cudaSuccess)
                return fail(MSC3D_ERR_CUDA);
            const double t_ready = ms_since();
            const unsigned long long ne = *hcnt;
            jp->n_esc = ne;
            cudaStream_t js = nullptr;
            if (cudaStreamCreateWithFlags(&js, cudaStreamNonBlocking) != cudaSuccess) return fail(MSC3D_ERR_CUDA);
            auto fetch = [&](void* h, const void* d, std::uint64_t bytes) {
                cudaError_t e = cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, js);
                if (e == cudaSuccess) e = cudaStreamSynchronize(js);
                return e == cudaSuccess;
            };
            if (ne > cap) {  // escapes did not fit: the full array itself
                const bool okf = fetch(host, dev, n * (kind == 0 ? 8 : 4));
                cudaStreamDestroy(js);
                jp->bytes = n * (kind == 0 ? 8 : 4);
                return okf ? void() : fail(MSC3D_ERR_CUDA);
            }
            const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
            const std::uint64_t T = n < (1ull << 20) ? 1 : std::min<std::uint64_t>(hw, 32);
            auto team = [&](auto f, std::uint64_t m, std::uint64_t nt) {
                std::vector<std::thread> ws;
                for (std::uint64_t k = 1; k < nt; ++k) ws.emplace_back(f, m * k / nt, m * (k + 1) / nt);
                f(0, m / nt);
                for (auto& w : ws) w.join();
            };
            // escapes beyond the speculative prefix (a first call, or a growing count)
            auto rest = [&]() { return ne <= guess || fetch(hesc + guess, desc + guess, (ne - guess) * 16); };
            double t_w1 = 0, t_e = 0;
            if (kind == 0) {
                auto* h64 = static_cast<std::uint64_t*>(host);
                // widen (no escape needed yet: it overlaps the block's other copies), then
                // patch the escaped entries (~1% random stores, split across threads)
                team([&](std::uint64_t a, std::uint64_t b) { msc3d_host::widen_u8_u64(h8, h64, a, b); }, n, T);
                t_w1 = ms_since();
                if (!rest()) return cudaStreamDestroy(js), fail(MSC3D_ERR_CUDA);
                t_e = ms_since();
                team([&](std::uint64_t a, std::uint64_t b) {
                    for (std::uint64_t k = a; k < b; ++k) h64[hesc[k].x] = hesc[k].y;
                }, ne, ne < (1ull << 16) ? 1 : T);
            } else {
                auto* h32 = static_cast<std::uint32_t*>(host);
                if (!rest()) return cudaStreamDestroy(js), fail(MSC3D_ERR_CUDA);
                t_e = ms_since();
                // escaped (absolute) values first, then every chunk from its head
                for (unsigned long long k = 0; k < ne; ++k) h32[hesc[k].x] = static_cast<std::uint32_t>(hesc[k].y);
                const std::uint64_t nch = (n + chunk - 1) / chunk;
                team([&](std::uint64_t c0, std::uint64_t c1) {
                    for (std::uint64_t c = c0; c < c1; ++c) {
                        const std::uint64_t a = c * chunk, b = std::min(n, a + chunk);
                        msc3d_host::decode_steps(h8, hheads[c], h32, a, b);
                    }
                    _mm_sfence();
                }, nch, std::min<std::uint64_t>(T, nch));
                t_w1 = ms_since();
            }
            cudaStreamDestroy(js);
            jp->bytes = ne > guess ? (ne - guess) * 16 : 0;
            if (dg)
                std::fprintf(stderr, "sink %s: %llu entries, bytes in at %.2f ms, escapes (%llu) by %.2f, decoded by "
                             "%.2f, done %.2f ms (host clock, %llu threads)\n", t.c_str(),
                             static_cast<unsigned long long>(n), t_ready, ne, t_e, t_w1, ms_since(),
                             static_cast<unsigned long long>(T));
        });
        jobs.push_back(std::move(job));
        return MSC3D_OK;
    }
    int finish() {
        int rc = MSC3D_OK;
        for (auto& j : jobs) {
            if (j->th.joinable()) j->th.join();
            if (j->rc != MSC3D_OK && rc == MSC3D_OK) rc = j->rc;
            bytes_moved += j->bytes;
            ctx->d2h_esc_memo[j->key] = j->n_esc;
        }
        jobs.clear();
        if (cs && cudaStreamSynchronize(cs) != cudaSuccess) rc = MSC3D_ERR_CUDA;
        if (diag && tl.size() >= 3) {
            cudaDeviceSynchronize();
            for (std::size_t k = 0; k + 2 < tl.size(); k += 3) {
                float r = 0, a = 0, b = 0;
                cudaEventElapsedTime(&r, tl[0], tl[k]);
                cudaEventElapsedTime(&a, tl[0], tl[k + 1]);
                cudaEventElapsedTime(&b, tl[0], tl[k + 2]);
                std::fprintf(stderr, "sink copy %zu: ready %.2f start %.2f end %.2f ms\n", k / 3, r, a, b);
            }
            for (std::size_t k = 0; k < tl.size(); k += 3) {
                cudaEventDestroy(tl[k + 1]);
                cudaEventDestroy(tl[k + 2]);
            }
            tl.clear();
        }
        for (auto e : evs) cudaEventDestroy(e);
        evs.clear();
        if (out) ctx->scalars["d2h_bytes"] = static_cast<std::int64_t>(bytes_moved);
        return rc;
    }
    ~Sink() { finish(); }
};

// The pipeline after the gradient.  forests_ready: parent0/parent3 already hold the
// extremum forests (the gradient kernel emits them); else they are built from the
// codes.  Sources: the critical 1-cells crit1[src_first, src_first + src_count) --
// all of them for a whole compute(); a slice when the saddle stages are sharded
// across GPUs (their 1s->2s arcs are then a contiguous block of the global list:
// "arcB_src/dst/mult").  grad_ms: the gradient's device time (already measured).
int compute_from_codes(msc3d_ctx* ctx, int options, double* stage_ms, const msc3d_host_outputs* host,
                       bool forests_ready, std::uint64_t src_first, std::uint64_t src_count, cudaEvent_t grad_t0,
                       bool sharded) {
    const Dims& d = ctx->dims;
    const int w = ctx->id_width();
    const cudaStream_t s = ctx->stream;
    const int sms = ctx->num_sms;
    const bool seg = (options & MSC3D_OPT_SEGMENTATION) != 0;
    StageClock clk(stage_ms != nullptr);
    Sink sink{ctx, host};
    clk.mark(0, s);
    cudaEvent_t t_start = nullptr;
    if (host && sink.diag) {
        cudaEventCreate(&t_start);
        cudaEventRecord(t_start, s);
    }

    clk.mark(1, s);

    // [critical] (multi-GPU: the per-slab lists, already gathered, multigpu.cu)
    if (ctx->crit_external) ctx->crit_external = false;
    else TRY(critical(ctx));
    clk.mark(2, s);
    const std::uint64_t c0 = ctx->scalars["c0"], c1 = ctx->scalars["c1"], c2 = ctx->scalars["c2"],
                        c3 = ctx->scalars["c3"];
    const std::uint64_t ncp = c0 + c1 + c2 + c3;
    if (ncp >= 0xffffffffull) return MSC3D_ERR_INVALID;  // cp ids are u32 (msc.hpp:25)
    ctx->decide_release(c1 + c2);
    const std::uint32_t base1 = static_cast<std::uint32_t>(c0), base2 = static_cast<std::uint32_t>(c0 + c1),
                        base3 = static_cast<std::uint32_t>(c0 + c1 + c2);

    // [extrema] roots by pointer jumping, saddle-extremum arcs, label remaps
    if (!forests_ready) {
        TRY(forest(ctx, 0));
        TRY(forest(ctx, 3));
    }
    {  // roots of both forests in place (the parent arrays become the label arrays)
        auto* flags = reinterpret_cast<unsigned int*>(ctx->d_small + 23);  // 3 x u32 (slots 23-24)
        auto* rounds = reinterpret_cast<unsigned long long*>(ctx->d_small + 25);
        MSC3D_CUDA_TRY(cudaMemsetAsync(ctx->d_small + 23, 0, 16, s));
        auto* conv = static_cast<unsigned int*>(
            ctx->ensure("jump_conv", (ctx->count("parent0") + ctx->count("parent3")) / 32 + 1, 4));
        if (!conv) return MSC3D_ERR_NOMEM;
        std::uint32_t* q0 = ctx->ptr<std::uint32_t>("parent0");
        std::uint32_t* q3 = ctx->ptr<std::uint32_t>("parent3");
        const std::uint64_t n0 = ctx->count("parent0"), n3 = ctx->count("parent3");
        // Long descending / ascending chains (big basins: few extrema per item, smooth
        // fields) are first resolved inside 32x16x16 boxes; the global jumping then only
        // chases the boxes' exit targets and one lookup finishes every other item.  With
        // small basins (noisy fields) the chains rarely leave a box and plain jumping is
        // cheaper than the extra passes.
        const bool tiled = (c0 + c3) * 64 < n0 + n3 && !std::getenv("MSC3D_NO_TILE_ROOTS");
        if (tiled) {
            MSC3D_CUDA_TRY(cudaMemsetAsync(conv, 0xff, ((n0 + n3) / 32 + 1) * 4, s));
            TRY(msc3d_dev::launch_tile_roots(q0, d.nx, d.ny, d.nz, conv, 0, flags + 3, s));
            TRY(msc3d_dev::launch_tile_roots(q3, d.nx - 1, d.ny - 1, d.nz - 1, conv, n0, flags + 3, s));
        }
        TRY(msc3d_dev::launch_jump_all(q0, n0, q3, n3, conv, flags, rounds, s, sms, tiled ? 1 : 0));
        if (tiled) TRY(msc3d_dev::launch_resolve_exits(q0, n0, q3, n3, s, sms));
    }
    auto* label0 = ctx->ptr<std::uint32_t>("parent0");
    auto* label3 = ctx->ptr<std::uint32_t>("parent3");
    // cp ids of the minima / maxima: bitmaps of the critical vertices / cubes with a
    // rank word per 32 entries (L2-resident) instead of full-size id maps
    msc3d_dev::RankRemap remap0{}, remap3{};
    {
        const std::uint64_t nw0 = d.n_verts / 32 + 1, nw3 = d.n_cubes / 32 + 1;
        const std::uint64_t nw = std::max(nw0, nw3);
        auto* bits = static_cast<unsigned int*>(ctx->ensure("rank_bits", nw, 4));
        auto* cnt = static_cast<std::uint32_t*>(ctx->ensure("rank_cnt", nw, 4));
        auto* pre = static_cast<std::uint64_t*>(ctx->ensure("rank_pre", nw, 8));
        auto* r0 = ctx->ensure("rank0", nw0, 8);
        auto* r3 = ctx->ensure("rank3", nw3, 8);
        if (!bits || !cnt || !pre || !r0 || !r3) return MSC3D_ERR_NOMEM;
        TRY(msc3d_dev::launch_rank_map(ctx->ptr<void>("crit0"), c0, w, d, 0, bits, cnt, pre, r0, nw0, ctx->ws,
                                       ctx->d_small + 38, s, sms));
        TRY(msc3d_dev::launch_rank_map(ctx->ptr<void>("crit3"), c3, w, d, 3, bits, cnt, pre, r3, nw3, ctx->ws,
                                       ctx->d_small + 38, s, sms));
        remap0 = msc3d_dev::RankRemap{static_cast<const uint2*>(r0), 0u};
        remap3 = msc3d_dev::RankRemap{static_cast<const uint2*>(r3), static_cast<std::uint32_t>(base3)};
    }
    // block A (min -> 1s) slots + per-minimum counts; block C (2s -> max) slots
    auto* slot_min = static_cast<std::uint32_t*>(ctx->ensure("slot_min", 2 * c1, 4));
    auto* per_min = static_cast<std::uint32_t*>(ctx->ensure("per_min", c0, 4));
    auto* min_off = static_cast<std::uint64_t*>(ctx->ensure("min_off", c0, 8));
    auto* slot_max = static_cast<std::uint32_t*>(ctx->ensure("slot_max", 2 * c2, 4));
    auto* cnt_max = static_cast<std::uint32_t*>(ctx->ensure("cnt_max", c2, 4));
    auto* off_max = static_cast<std::uint64_t*>(ctx->ensure("off_max", c2, 8));
    if (!slot_min || !per_min || !min_off || !slot_max || !cnt_max || !off_max) return MSC3D_ERR_NOMEM;
    if (c0) MSC3D_CUDA_TRY(cudaMemsetAsync(per_min, 0, c0 * 4, s));
    TRY(msc3d_dev::launch_arcs_min(ctx->ptr<void>("crit1"), c1, w, d, label0, remap0, base1, slot_min,
                                   per_min, s, sms));
    TRY(msc3d_dev::launch_arcs_max(ctx->ptr<void>("crit2"), c2, w, d, label3, remap3, slot_max, cnt_max, s, sms));
    TRY(msc3d_dev::scan_u32(per_min, c0, min_off, ctx->d_small + 32, ctx->ws, s));
    TRY(msc3d_dev::scan_u32(cnt_max, c2, off_max, ctx->d_small + 33, ctx->ws2, s));
    clk.mark(3, s);

    // ---- outputs that are final now (untimed in the reference's StageTimings) ----
    // critical points, label volumes, min->1s and 2s->max arcs; their host copies
    // overlap the saddle stages
    TRY(ctx->fetch_small(34));
    // root finding did not converge (globally, or inside a box): a cycle
    if (ctx->h_small[25] > 64 || (ctx->h_small[24] >> 32)) return MSC3D_ERR_RUNTIME;
    ctx->scalars["jump_rounds"] = static_cast<std::int64_t>(ctx->h_small[25]);
    const std::uint64_t na = c0 ? ctx->h_small[32] : 0;  // min->1s arcs
    const std::uint64_t nc = c2 ? ctx->h_small[33] : 0;  // 2s->max arcs
    ctx->scalars["arcs_min"] = static_cast<std::int64_t>(na);
    ctx->scalars["arcs_max"] = static_cast<std::int64_t>(nc);
    void* cp_cell = ctx->ensure("cp_cell", ncp, w);
    auto* cp_index = static_cast<std::uint8_t*>(ctx->ensure("cp_index", ncp, 1));
    // A whole compute() writes the min->1s block straight into the final arc arrays (it
    // leads them), sized by the previous call's 1s->2s count (or 4 per 1-saddle) and
    // grown keeping it if the count turns out larger; a 1-saddle slice keeps it apart.
    const bool a_in_place = !(sharded ? src_count > 1
                                      : (src_first != 0 || src_first > c1 ||
                                         std::min<std::uint64_t>(src_count, c1 - src_first) != c1));
    std::uint64_t nb_guess = 4 * c1;
    if (auto it = ctx->scalars.find("arcs_ss"); it != ctx->scalars.end()) nb_guess = static_cast<std::uint64_t>(it->second);
    const std::uint64_t a_cap = na + nb_guess + nc;
    auto* amin_src = static_cast<std::uint32_t*>(a_in_place ? ctx->ensure("arc_src", a_cap, 4) : ctx->ensure("arcA_src", na, 4));
    auto* amin_dst = static_cast<std::uint32_t*>(a_in_place ? ctx->ensure("arc_dst", a_cap, 4) : ctx->ensure("arcA_dst", na, 4));
    auto* amin_mul = static_cast<std::uint64_t*>(a_in_place ? ctx->ensure("arc_mult", a_cap, 8) : ctx->ensure("arcA_mult", na, 8));
    if (a_in_place) {
        ctx->drop("arcA_src");
        ctx->drop("arcA_dst");
        ctx->drop("arcA_mult");
    }
    auto* amax_src = static_cast<std::uint32_t*>(ctx->ensure("arcC_src", nc, 4));
    auto* amax_dst = static_cast<std::uint32_t*>(ctx->ensure("arcC_dst", nc, 4));
    auto* amax_mul = static_cast<std::uint64_t*>(ctx->ensure("arcC_mult", nc, 8));
    auto* key = static_cast<std::uint64_t*>(ctx->ensure("sort_key", na, 8));
    auto* scratch = static_cast<std::uint64_t*>(ctx->ensure("sort_scratch", na, 8));
    auto* cursor = static_cast<std::uint32_t*>(ctx->ensure("sort_cursor", c0, 4));
    auto* large = static_cast<std::uint32_t*>(ctx->ensure("sort_large", c0, 4));
    if (!cp_cell || !cp_index || !amin_src || !amin_dst || !amin_mul || !amax_src || !amax_dst || !amax_mul || !key ||
        !scratch || !cursor || !large)
        return MSC3D_ERR_NOMEM;
    // Option "side_stream": the assembly of the extremum-side outputs (critical point
    // list, label volumes, sorted min->1s and 2s->max arcs: ~3 ms of small
    // bandwidth-bound kernels, no host round trips) runs on a side stream, beside the
    // latency-bound saddle stages; the main stream waits for it before it touches those
    // arrays (Join, at every exit).  Measured at 512^3: the step gains 0.3 ms, but the
    // saddle stages slow down by ~2.3 ms under the contention, which blurs the
    // per-stage timings -- off by default.  (Grids above 2^32 cells free scratch
    // mid-way: they keep one stream.)
    const cudaStream_t sa = ctx->release_transients() || !ctx->side_assembly ? s : ctx->side_stream();
    if (!sa) return MSC3D_ERR_CUDA;
    struct Join {
        cudaStream_t main, side;
        cudaEvent_t ev = nullptr;
        ~Join() {
            if (!ev) return;
            cudaEventRecord(ev, side);
            cudaStreamWaitEvent(main, ev, 0);
            cudaEventDestroy(ev);
        }
    } join{s, sa};
    if (sa != s) {
        cudaEvent_t fork;
        MSC3D_CUDA_TRY(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
        MSC3D_CUDA_TRY(cudaEventRecord(fork, s));
        MSC3D_CUDA_TRY(cudaStreamWaitEvent(sa, fork, 0));
        cudaEventDestroy(fork);
        MSC3D_CUDA_TRY(cudaEventCreateWithFlags(&join.ev, cudaEventDisableTiming));
    }
    sink.producer = sa;
    std::uint64_t at = 0;
    for (int k = 0; k < 4; ++k) {
        const std::string nm = "crit" + std::to_string(k);
        const std::uint64_t n = ctx->count(nm);
        TRY(msc3d_dev::launch_cp_concat(ctx->ptr<void>(nm), n, at, k, w, cp_cell, cp_index, sa, sms));
        at += n;
    }
    if (host) {
        if (host->cp_cell_cap < ncp * w || host->cp_index_cap < ncp) return MSC3D_ERR_INVALID;
        TRY(sink.copy(host->cp_cell, cp_cell, ncp * w));
        TRY(sink.copy(host->cp_index, cp_index, ncp));
    }
    if (seg) {
        auto* lmin = static_cast<std::uint32_t*>(ctx->ensure("labels_min", d.n_verts, 4));
        auto* lmax = static_cast<std::uint32_t*>(ctx->ensure("labels_max", d.n_cubes, 4));
        if (!lmin || (!lmax && d.n_cubes)) return MSC3D_ERR_NOMEM;
        TRY(msc3d_dev::launch_gather(label0, remap0, d.n_verts, lmin, sa, sms));
        TRY(msc3d_dev::launch_gather(label3, remap3, d.n_cubes, lmax, sa, sms));
        if (host) {
            TRY(sink.copy(host->labels_min, lmin, d.n_verts * 4));
            TRY(sink.copy(host->labels_max, lmax, d.n_cubes * 4));
        }
    } else {
        ctx->drop("labels_min");
        ctx->drop("labels_max");
    }
    TRY(msc3d_dev::launch_arcs_min_sort(slot_min, c1, base1, min_off, c0, na, cursor, key, scratch, large,
                                        reinterpret_cast<unsigned long long*>(ctx->d_small + 35),
                                        ctx->h_small + 35, amin_src, amin_dst, amin_mul, sa, sms));
    TRY(msc3d_dev::launch_arcs_max_emit(slot_max, c2, base2, off_max, amax_src, amax_dst, amax_mul, sa, sms));
    if (ctx->release_transients())
        for (const char* t : {"slot_min", "per_min", "min_off", "slot_max", "cnt_max", "off_max", "sort_key",
                              "sort_scratch", "sort_cursor", "sort_large", "rank_bits", "rank_cnt", "rank_pre",
                              "star_list16", "star_list32", "star_list_ties", "jump_conv"})
            ctx->release(t);
    if (host) {
        if (host->arc_cap < na) return MSC3D_ERR_INVALID;
        // (the multiplicity bytes first: their host widening overlaps the other copies)
        TRY(sink.copy_mult(host->arc_mult, amin_mul, na, "A"));
        TRY(sink.copy_src(host->arc_src, amin_src, na, "A"));
        TRY(sink.copy(host->arc_dst, amin_dst, na * 4));
    }
    sink.producer = nullptr;
    clk.mark(4, s);  // (end of the untimed block: re-based below)

    // [reachability]
    StageClock clk2(stage_ms != nullptr);
    clk2.mark(0, s);
    std::uint64_t n_shards = 1;
    if (sharded) {  // shard src_first of src_count balanced slices
        const std::uint64_t k = src_first, n = src_count;
        n_shards = n;
        src_first = c1 * k / n;
        src_count = c1 * (k + 1) / n - src_first;
        ctx->scalars["shard_first"] = static_cast<std::int64_t>(src_first);
        ctx->scalars["shard_count"] = static_cast<std::int64_t>(src_count);
    }
    if (src_first > c1) return MSC3D_ERR_INVALID;
    src_count = std::min(src_count, c1 - src_first);
    // a rank of a multi-shard run always delivers its block in arcB_* (even when the
    // balanced slice happens to be empty or the whole list)
    const bool sliced = sharded ? n_shards > 1 : (src_first != 0 || src_count != c1);
    const void* srcs = static_cast<const char*>(ctx->ptr<void>("crit1")) + src_first * w;
    TRY(bfs(ctx, srcs, src_count));
    clk2.mark(1, s);

    // [counting] -- 1s->2s arcs written straight into the final arc arrays (as cp ids)
    std::uint32_t *asrc = nullptr, *adst = nullptr;
    std::uint64_t* amul = nullptr;
    auto place = [&](std::uint64_t nb, CountOut* o) -> int {
        if (sliced) {  // this shard's block only
            o->one = static_cast<std::uint32_t*>(ctx->ensure("arcB_src", nb, 4));
            o->two = static_cast<std::uint32_t*>(ctx->ensure("arcB_dst", nb, 4));
            o->paths = static_cast<std::uint64_t*>(ctx->ensure("arcB_mult", nb, 8));
            o->base_one = base1 + static_cast<std::uint32_t>(src_first);
            o->base_two = base2;
            return MSC3D_OK;
        }
        const std::uint64_t total = na + nb + nc;
        const std::uint64_t keep = a_in_place ? na : 0;  // (the min->1s block already in place)
        asrc = static_cast<std::uint32_t*>(ctx->ensure_keep("arc_src", total, 4, keep * 4, s));
        adst = static_cast<std::uint32_t*>(ctx->ensure_keep("arc_dst", total, 4, keep * 4, s));
        amul = static_cast<std::uint64_t*>(ctx->ensure_keep("arc_mult", total, 8, keep * 8, s));
        if (!asrc || !adst || !amul) return MSC3D_ERR_NOMEM;
        if (host) {  // the 2s->max block's host position is known now: send it before the 1s->2s block
            if (host->arc_cap < total) return MSC3D_ERR_INVALID;
            sink.producer = sa;  // (produced on the side stream)
            TRY(sink.copy_mult(host->arc_mult + na + nb, amax_mul, nc, "C"));
            TRY(sink.copy_src(host->arc_src + na + nb, amax_src, nc, "C"));
            TRY(sink.copy(host->arc_dst + na + nb, amax_dst, nc * 4));
            sink.producer = nullptr;
        }
        o->one = asrc + na;
        o->two = adst + na;
        o->paths = amul + na;
        o->base_one = base1;
        o->base_two = base2;
        return MSC3D_OK;
    };
    TRY(dag_count(ctx, srcs, src_count, "crit2", place));
    clk2.mark(2, s);
    const std::uint64_t nb = static_cast<std::uint64_t>(ctx->scalars["arcs_ss"]);
    if (sliced) {
        if (host) return MSC3D_ERR_INVALID;  // host delivery is for whole computes
        ctx->drop("arc_src");
        ctx->drop("arc_dst");
        ctx->drop("arc_mult");
        if (stage_ms) {
            MSC3D_CUDA_TRY(cudaStreamSynchronize(s));
            for (int i = 0; i < 3; ++i) {
                float ms = 0;
                if (clk.ok) cudaEventElapsedTime(&ms, i == 0 && grad_t0 ? grad_t0 : clk.ev[i], clk.ev[i + 1]);
                stage_ms[i] = ms;
            }
            for (int i = 0; i < 2; ++i) {
                float ms = 0;
                if (clk2.ok) cudaEventElapsedTime(&ms, clk2.ev[i], clk2.ev[i + 1]);
                stage_ms[3 + i] = ms;
            }
        }
        return MSC3D_OK;
    }
    if (host) {
        if (host->arc_cap < na + nb + nc) return MSC3D_ERR_INVALID;
        TRY(sink.copy_mult(host->arc_mult + na, amul + na, nb, "B"));
        TRY(sink.copy_src(host->arc_src + na, asrc + na, nb, "B"));
        TRY(sink.copy(host->arc_dst + na, adst + na, nb * 4));
    }
    // device-side arc arrays complete: the min and max blocks around the 1s->2s block
    if (join.ev) {  // (the side stream's arrays: wait for them here already)
        MSC3D_CUDA_TRY(cudaEventRecord(join.ev, sa));
        MSC3D_CUDA_TRY(cudaStreamWaitEvent(s, join.ev, 0));
    }
    if (na && !a_in_place) {
        MSC3D_CUDA_TRY(cudaMemcpyAsync(asrc, amin_src, na * 4, cudaMemcpyDeviceToDevice, s));
        MSC3D_CUDA_TRY(cudaMemcpyAsync(adst, amin_dst, na * 4, cudaMemcpyDeviceToDevice, s));
        MSC3D_CUDA_TRY(cudaMemcpyAsync(amul, amin_mul, na * 8, cudaMemcpyDeviceToDevice, s));
    }
    if (nc) {
        MSC3D_CUDA_TRY(cudaMemcpyAsync(asrc + na + nb, amax_src, nc * 4, cudaMemcpyDeviceToDevice, s));
        MSC3D_CUDA_TRY(cudaMemcpyAsync(adst + na + nb, amax_dst, nc * 4, cudaMemcpyDeviceToDevice, s));
        MSC3D_CUDA_TRY(cudaMemcpyAsync(amul + na + nb, amax_mul, nc * 8, cudaMemcpyDeviceToDevice, s));
    }
    if (host && sink.diag && t_start) {
        cudaEvent_t t_end;
        cudaEventCreate(&t_end);
        cudaEventRecord(t_end, s);
        cudaEventSynchronize(t_end);
        float a = 0, b = 0;
        if (!sink.tl.empty()) cudaEventElapsedTime(&a, t_start, sink.tl[0]);
        cudaEventElapsedTime(&b, t_start, t_end);
        std::fprintf(stderr, "pipeline: first copy ready at %.2f ms, compute stream done at %.2f ms\n", a, b);
        cudaEventDestroy(t_end);
        cudaEventDestroy(t_start);
    }
    if (host) {
        auto* h = const_cast<msc3d_host_outputs*>(host);
        h->n_cp = ncp;
        h->n_arcs = na + nb + nc;
        TRY(sink.finish());
    }
    if (stage_ms) {
        MSC3D_CUDA_TRY(cudaStreamSynchronize(s));
        for (int i = 0; i < 3; ++i) {
            float ms = 0;
            if (clk.ok) cudaEventElapsedTime(&ms, i == 0 && grad_t0 ? grad_t0 : clk.ev[i], clk.ev[i + 1]);
            stage_ms[i] = ms;
        }
        for (int i = 0; i < 2; ++i) {
            float ms = 0;
            if (clk2.ok) cudaEventElapsedTime(&ms, clk2.ev[i], clk2.ev[i + 1]);
            stage_ms[3 + i] = ms;
        }
    }
    return MSC3D_OK;
}

int validate(msc3d_ctx* ctx);

// The whole pipeline from HOST samples: the input goes up in z-chunks on a copy
// stream and the gradient's tile layers start as soon as the planes they read have
// arrived, so the upload overlaps the gradient; the outputs come back as in
// compute_host.  Non-finite samples -> invalid_argument (grid.cpp:86-88), checked
// on the device after the upload.
int compute_streamed(msc3d_ctx* ctx, const void* host_values, int value_type, int options, double* stage_ms,
                     const msc3d_host_outputs* host) {
    const Dims& d = ctx->dims;
    const int elem = value_type == MSC3D_VALUE_F64 ? 8 : 4;
    void* vals = ctx->ensure("values", d.n_verts, elem);
    if (!vals) return MSC3D_ERR_NOMEM;
    ctx->values = vals;
    ctx->value_type = value_type;
    const cudaStream_t s = ctx->stream;
    const cudaStream_t up = ctx->h2d_stream();
    if (!up) return MSC3D_ERR_CUDA;
    cudaEvent_t t0 = nullptr;
    if (stage_ms) {
        MSC3D_CUDA_TRY(cudaEventCreate(&t0));
        MSC3D_CUDA_TRY(cudaEventRecord(t0, s));
        MSC3D_CUDA_TRY(cudaStreamWaitEvent(up, t0, 0));
    }
    // chunks of vertex planes
    const std::uint64_t plane = static_cast<std::uint64_t>(d.nx) * d.ny * elem;
    std::int64_t chunk_bytes = 32ll << 20;  // ~32 MB per upload chunk (MSC3D_UPLOAD_CHUNK_KB overrides, for tests)
    if (const char* e = std::getenv("MSC3D_UPLOAD_CHUNK_KB")) chunk_bytes = std::max(1ll, std::atoll(e)) << 10;
    const std::int64_t zc = std::max<std::int64_t>(2, chunk_bytes / static_cast<std::int64_t>(plane));
    const std::int64_t nchunks = (d.nz + zc - 1) / zc;
    std::vector<cudaEvent_t> ev(static_cast<std::size_t>(nchunks), nullptr);
    int rc = MSC3D_OK;
    for (std::int64_t c = 0; c < nchunks && rc == MSC3D_OK; ++c) {
        const std::int64_t z0 = c * zc, z1 = std::min<std::int64_t>(d.nz, z0 + zc);
        if (cudaMemcpyAsync(static_cast<char*>(vals) + z0 * plane, static_cast<const char*>(host_values) + z0 * plane,
                            (z1 - z0) * plane, cudaMemcpyHostToDevice, up) != cudaSuccess ||
            cudaEventCreateWithFlags(&ev[c], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventRecord(ev[c], up) != cudaSuccess)
            rc = MSC3D_ERR_CUDA;
    }
    auto cleanup = [&]() {
        for (auto e : ev)
            if (e) cudaEventDestroy(e);
        if (t0) cudaEventDestroy(t0);
    };
    // gradient tile layers as their planes arrive
    auto* codes = static_cast<std::uint8_t*>(ctx->ensure("codes", d.n_cells, 1));
    auto* p0 = static_cast<std::uint32_t*>(ctx->ensure("parent0", d.n_verts, 4));
    auto* p3 = static_cast<std::uint32_t*>(ctx->ensure("parent3", d.n_cubes, 4));
    std::uint32_t* lists[3] = {static_cast<std::uint32_t*>(ctx->ensure("star_list16", 2 * d.n_verts, 4)),
                               static_cast<std::uint32_t*>(ctx->ensure("star_list32", 2 * d.n_verts, 4)),
                               static_cast<std::uint32_t*>(ctx->ensure("star_list_ties", d.n_verts, 4))};
    if (!codes || !p0 || !p3 || !lists[0] || !lists[1] || !lists[2]) rc = rc ? rc : MSC3D_ERR_NOMEM;
    auto* crit_totals = reinterpret_cast<unsigned long long*>(ctx->d_small + 40);
    auto* list_counts = reinterpret_cast<unsigned long long*>(ctx->d_small + 44);
    if (rc == MSC3D_OK) rc = msc3d_dev::gradient_begin(crit_totals, list_counts, s);
    const unsigned layers = msc3d_dev::gradient_tile_layers(d);
    const unsigned step = static_cast<unsigned>(std::max<std::int64_t>(1, zc / 2));
    std::int64_t waited = -1;
    for (unsigned t0l = 0; t0l < layers && rc == MSC3D_OK; t0l += step) {
        const unsigned t1l = std::min(layers, t0l + step);
        const std::int64_t need = msc3d_dev::gradient_layer_last_plane(d, t1l) / zc;  // chunk of the last plane read
        for (; waited < need && rc == MSC3D_OK; ++waited)
            if (cudaStreamWaitEvent(s, ev[waited + 1], 0) != cudaSuccess) rc = MSC3D_ERR_CUDA;
        if (rc == MSC3D_OK)
            rc = msc3d_dev::gradient_tiles(vals, value_type, d, codes, p0, p3, s, crit_totals, lists, list_counts,
                                           ctx->num_sms, t0l, t1l);
    }
    for (; waited + 1 < nchunks && rc == MSC3D_OK; ++waited)
        if (cudaStreamWaitEvent(s, ev[waited + 1], 0) != cudaSuccess) rc = MSC3D_ERR_CUDA;
    if (rc == MSC3D_OK)
        rc = msc3d_dev::gradient_finish(vals, value_type, d, codes, p0, p3, s, crit_totals, lists, list_counts,
                                        ctx->num_sms);
    // samples must be finite (checked once all of them are up)
    auto* bad = reinterpret_cast<unsigned long long*>(ctx->d_small + 22);
    if (rc == MSC3D_OK && cudaMemsetAsync(bad, 0xff, 8, s) != cudaSuccess) rc = MSC3D_ERR_CUDA;
    if (rc == MSC3D_OK) rc = msc3d_dev::launch_check_finite(vals, value_type, d.n_verts, bad, s, ctx->num_sms);
    if (rc == MSC3D_OK) rc = ctx->fetch_range(22, 1);
    if (rc == MSC3D_OK && ctx->h_small[22] != ~0ull) rc = MSC3D_ERR_INVALID;
    ctx->crit_counts_valid = true;
    if (rc == MSC3D_OK && (options & MSC3D_OPT_VALIDATE)) rc = validate(ctx);
    if (rc == MSC3D_OK) rc = compute_from_codes(ctx, options, stage_ms, host, true, 0, ~0ull, t0);
    cleanup();
    return rc;
}

// ComputeOptions::validate (msc.cpp:67-70): validate_gradient with the reference's
// default cycle-check bound (gradient.hpp:95-96) on the device; a broken gradient ->
// runtime_error.
int validate(msc3d_ctx* ctx) {
    std::uint64_t r[4];
    TRY(audit_gradient(ctx, 100000, r));
    ctx->scalars["validate_violations"] = static_cast<std::int64_t>(r[0]);
    ctx->scalars["validate_closed_vpath_cells"] = static_cast<std::int64_t>(r[1]);
    return (r[0] || r[1]) ? MSC3D_ERR_RUNTIME : MSC3D_OK;
}

// The outputs of the last computation (device arrays of the context) delivered to host
// buffers the way compute_host does: multiplicities and sorted sources narrow, decoded
// by host threads, the rest copied.  For results computed device-resident (e.g. by the
// multi-GPU step) that are wanted on the host afterwards.
int deliver_host(msc3d_ctx* ctx, const msc3d_host_outputs* host) {
    for (const char* nm : {"cp_cell", "cp_index", "arc_src", "arc_dst", "arc_mult"})
        if (!ctx->find(nm)) return MSC3D_ERR_STATE;
    const std::uint64_t ncp = ctx->count("cp_index"), na = ctx->count("arc_src");
    const int w = ctx->id_width();
    if (host->cp_cell_cap < ncp * w || host->cp_index_cap < ncp || host->arc_cap < na) return MSC3D_ERR_INVALID;
    Sink sink{ctx, host};
    TRY(sink.copy(host->cp_cell, ctx->ptr<void>("cp_cell"), ncp * w));
    TRY(sink.copy(host->cp_index, ctx->ptr<void>("cp_index"), ncp));
    if (host->labels_min && ctx->find("labels_min") && ctx->count("labels_min"))
        TRY(sink.copy(host->labels_min, ctx->ptr<void>("labels_min"), ctx->count("labels_min") * 4));
    if (host->labels_max && ctx->find("labels_max") && ctx->count("labels_max"))
        TRY(sink.copy(host->labels_max, ctx->ptr<void>("labels_max"), ctx->count("labels_max") * 4));
    TRY(sink.copy_mult(host->arc_mult, ctx->ptr<std::uint64_t>("arc_mult"), na, "X"));
    TRY(sink.copy_src(host->arc_src, ctx->ptr<std::uint32_t>("arc_src"), na, "X"));
    TRY(sink.copy(host->arc_dst, ctx->ptr<void>("arc_dst"), na * 4));
    auto* h = const_cast<msc3d_host_outputs*>(host);
    h->n_cp = ncp;
    h->n_arcs = na;
    return sink.finish();
}

int compute(msc3d_ctx* ctx, int options, double* stage_ms, const msc3d_host_outputs* host) {
    // [gradient] codes + both extremum forests in one kernel
    cudaEvent_t t0 = nullptr;
    if (stage_ms) {
        MSC3D_CUDA_TRY(cudaEventCreate(&t0));
        MSC3D_CUDA_TRY(cudaEventRecord(t0, ctx->stream));
    }
    int rc = gradient(ctx, /*with_forests=*/true);
    if (rc == MSC3D_OK && (options & MSC3D_OPT_VALIDATE)) rc = validate(ctx);
    if (rc == MSC3D_OK)
        rc = compute_from_codes(ctx, options, stage_ms, host, true, 0, ~0ull, t0);
    if (t0) cudaEventDestroy(t0);
    return rc;
}

}  // namespace msc3d_stage

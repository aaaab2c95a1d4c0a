// Device audits of a gradient and of an assembled complex:
//
// * validate_gradient (proj/src/gradient.cpp:299-377): the matching audit over all
//   cells (every paired cell's partner exists, has the dimension one up / down and
//   points back), then -- for grids up to max_cells_for_cycles cells, as the reference
//   -- acyclicity of the V-path relation "alpha -> other facets of alpha's cofacet
//   partner that are themselves paired upward", by Kahn peeling: an in-degree pass,
//   then one cooperative kernel that peels frontier after frontier with a grid barrier
//   per level.  Whatever is never peeled sits on a closed V-path.
// * boundary_check (proj/src/msc.cpp:149-167): for every critical point t of index 2
//   or 3, the mod-2 sum over two-step descents t <- mid <- low of m(mid,t)*m(low,mid)
//   must vanish for every low.  Arcs are bucketed by destination (counting sort), each
//   top's odd-odd two-step toggles are listed, sorted per top and run-length parity
//   counted; the odd (top, low) pairs come out in the reference's order (tops by id,
//   lows ascending).
#include <cooperative_groups.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "ctx.cuh"
#include "kernels.cuh"
#include "stages.cuh"

namespace cg = cooperative_groups;

namespace msc3d_dev {
namespace {

constexpr int kT = 256;
constexpr int kSampleCap = 4096;

inline unsigned blocks_for(std::uint64_t n) {
    return static_cast<unsigned>(std::max<std::uint64_t>(1, std::min<std::uint64_t>((n + kT - 1) / kT, 1u << 20)));
}

#define AUDIT_STRIDE(i, n)                                                                        \
    for (std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x; \
         i < (n); i += static_cast<std::uint64_t>(gridDim.x) * blockDim.x)

// one slot per calling lane on a global counter, one atomic per warp
__device__ __forceinline__ unsigned long long claim(unsigned long long* ctr) {
    cg::coalesced_group g = cg::coalesced_threads();
    unsigned long long base = 0;
    if (g.thread_rank() == 0) base = atomicAdd(ctr, static_cast<unsigned long long>(g.size()));
    return g.shfl(base, 0) + g.thread_rank();
}

// stats: [0] violations [1] pairs [2] samples recorded
__global__ void k_matching(const std::uint8_t* __restrict__ codes, Dims d, unsigned long long* stats,
                           std::uint64_t* samples) {
    unsigned long long bad = 0, pairs = 0;
    const std::int64_t step[3] = {1, d.ex, d.exy};
    const std::int64_t ext[3] = {d.ex, d.ey, d.ez};
    AUDIT_STRIDE(c, d.n_cells) {
        const std::uint8_t k = codes[c];
        if (k == kCritical) continue;
        bool ok = k != kUnset && k < kCofacetBase + 6;
        if (ok) {
            ++pairs;
            const bool up = k >= kCofacetBase;
            const int dir = k - (up ? kCofacetBase : kFacetBase), axis = dir >> 1;
            const std::int64_t sign = (dir & 1) ? 1 : -1;
            const Coord cc = unpack(d, c);
            const std::int64_t co = axis == 0 ? cc.x : (axis == 1 ? cc.y : cc.z);
            // a cofacet partner lies along an even axis, a facet partner along an odd one
            ok = ((co & 1) == 0) == up && co + sign >= 0 && co + sign < ext[axis];
            if (ok) {
                const std::uint8_t back = static_cast<std::uint8_t>((up ? kFacetBase : kCofacetBase) + axis * 2 +
                                                                    (sign > 0 ? 0 : 1));
                ok = codes[c + sign * step[axis]] == back;
            }
        }
        if (!ok) {
            ++bad;
            const unsigned long long at = claim(&stats[2]);
            if (at < kSampleCap) samples[at] = c;
        }
    }
    for (int o = 16; o; o >>= 1) {
        bad += __shfl_xor_sync(0xffffffffu, bad, o);
        pairs += __shfl_xor_sync(0xffffffffu, pairs, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (bad) atomicAdd(&stats[0], bad);
        if (pairs) atomicAdd(&stats[1], pairs);
    }
}

// V-path successors of an upward-paired cell c (gradient.cpp:341-350): the facets x
// of b = partner(c) other than c that are paired upward.  Facets of b step along
// b's odd axes, so they always lie inside the box.
template <typename F>
__device__ __forceinline__ void for_each_next(const std::uint8_t* __restrict__ codes, const Dims& d,
                                              std::uint64_t c, std::uint8_t k, F&& f) {
    if (k >= kCofacetBase + 6) return;  // malformed: counted by the matching audit
    const std::int64_t b = partner_of(d, static_cast<std::int64_t>(c), k);
    if (b < 0 || static_cast<std::uint64_t>(b) >= d.n_cells) return;
    const Coord cb = unpack(d, static_cast<std::uint64_t>(b));
    const std::int64_t co[3] = {cb.x, cb.y, cb.z};
    const std::int64_t step[3] = {1, d.ex, d.exy};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        if (!(co[a] & 1)) continue;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const std::int64_t x = b + (h ? step[a] : -step[a]);
            if (static_cast<std::uint64_t>(x) != c && codes[x] >= kCofacetBase) f(static_cast<std::uint64_t>(x));
        }
    }
}

// in-degrees of the V-path relation; stats[3] = upward-paired cells
__global__ void k_vpath_indeg(const std::uint8_t* __restrict__ codes, Dims d, std::uint32_t* __restrict__ indeg,
                              unsigned long long* stats) {
    unsigned long long up = 0;
    AUDIT_STRIDE(c, d.n_cells) {
        const std::uint8_t k = codes[c];
        if (k < kCofacetBase) continue;
        ++up;
        for_each_next(codes, d, c, k, [&](std::uint64_t x) { atomicAdd(&indeg[x], 1u); });
    }
    for (int o = 16; o; o >>= 1) up += __shfl_xor_sync(0xffffffffu, up, o);
    if ((threadIdx.x & 31) == 0 && up) atomicAdd(&stats[3], up);
}

__global__ void k_vpath_seed(const std::uint8_t* __restrict__ codes, Dims d, const std::uint32_t* __restrict__ indeg,
                             std::uint64_t* __restrict__ frontier, unsigned long long* cnt) {
    AUDIT_STRIDE(c, d.n_cells) {
        if (codes[c] >= kCofacetBase && indeg[c] == 0) frontier[claim(&cnt[0])] = c;
    }
}

// Kahn peeling, all levels in one cooperative launch.  Frontier sizes rotate over
// cnt[0..2]: level L reads cnt[L%3], appends to cnt[(L+1)%3] and clears cnt[(L+2)%3]
// (read at level L-1, written at level L+1: untouched during level L).  cnt[0] holds
// the seed frontier size, cnt[1] = cnt[2] = 0; cnt[3] accumulates peeled cells,
// cnt[4] receives the level count.
__global__ void __launch_bounds__(kT) k_vpath_peel(const std::uint8_t* __restrict__ codes, Dims d,
                                                   std::uint32_t* __restrict__ indeg, std::uint64_t* fa,
                                                   std::uint64_t* fb, unsigned long long* cnt) {
    cg::grid_group grid = cg::this_grid();
    std::uint64_t* cur = fa;
    std::uint64_t* nxt = fb;
    for (int level = 0;; ++level) {
        const unsigned long long n = *reinterpret_cast<volatile unsigned long long*>(&cnt[level % 3]);
        if (n == 0) {
            if (grid.thread_rank() == 0) cnt[4] = static_cast<unsigned long long>(level);
            break;
        }
        AUDIT_STRIDE(i, n) {
            const std::uint64_t c = cur[i];
            for_each_next(codes, d, c, codes[c], [&](std::uint64_t x) {
                if (atomicSub(&indeg[x], 1u) == 1u) nxt[claim(&cnt[(level + 1) % 3])] = x;
            });
        }
        if (grid.thread_rank() == 0) {
            cnt[3] += n;
            cnt[(level + 2) % 3] = 0;
        }
        grid.sync();
        std::uint64_t* t = cur;
        cur = nxt;
        nxt = t;
    }
}

// ---- boundary check ----------------------------------------------------------------

__global__ void k_in_count(const std::uint32_t* __restrict__ dst, std::uint64_t n, std::uint32_t* __restrict__ cnt) {
    AUDIT_STRIDE(i, n) atomicAdd(&cnt[dst[i]], 1u);
}

__global__ void k_in_fill(const std::uint32_t* __restrict__ dst, std::uint64_t n, const std::uint64_t* __restrict__ off,
                          std::uint32_t* __restrict__ cursor, std::uint64_t* __restrict__ in_arc) {
    AUDIT_STRIDE(i, n) {
        const std::uint32_t t = dst[i];
        in_arc[off[t] + atomicAdd(&cursor[t], 1u)] = i;
    }
}

// pass 0: count the top's odd-odd two-step toggles; pass 1: write them
template <bool kWrite>
__global__ void k_toggles(const std::uint8_t* __restrict__ cp_index, std::uint64_t n_cp,
                          const std::uint32_t* __restrict__ src, const std::uint64_t* __restrict__ mult,
                          const std::uint64_t* __restrict__ in_off, const std::uint32_t* __restrict__ in_cnt,
                          const std::uint64_t* __restrict__ in_arc, std::uint32_t* __restrict__ tcnt,
                          const std::uint64_t* __restrict__ toff, std::uint32_t* __restrict__ tbuf,
                          unsigned int* __restrict__ too_many) {
    AUDIT_STRIDE(t, n_cp) {
        if (cp_index[t] < 2) {
            if (!kWrite) tcnt[t] = 0;
            continue;
        }
        std::uint64_t k = 0;
        const std::uint64_t b0 = in_off[t], e0 = b0 + in_cnt[t];
        for (std::uint64_t a = b0; a < e0; ++a) {
            const std::uint64_t arc = in_arc[a];
            if (!(mult[arc] & 1u)) continue;
            const std::uint32_t mid = src[arc];
            const std::uint64_t b1 = in_off[mid], e1 = b1 + in_cnt[mid];
            for (std::uint64_t a2 = b1; a2 < e1; ++a2) {
                const std::uint64_t arc2 = in_arc[a2];
                if (!(mult[arc2] & 1u)) continue;
                if (kWrite) tbuf[toff[t] + k] = src[arc2];
                ++k;
            }
        }
        if (!kWrite) {
            if (k > 0xffffffffull) *too_many = 1u;
            tcnt[t] = static_cast<std::uint32_t>(k);
        }
    }
}

// Sort each top's toggles (insertion sort in place: segments are short), keep the
// lows that occur an odd number of times, packed at the segment start.
__global__ void k_toggle_parity(std::uint64_t n_cp, const std::uint64_t* __restrict__ toff,
                                const std::uint32_t* __restrict__ tcnt, std::uint32_t* __restrict__ tbuf,
                                std::uint32_t* __restrict__ ocnt) {
    AUDIT_STRIDE(t, n_cp) {
        std::uint32_t* s = tbuf + toff[t];
        const std::uint32_t n = tcnt[t];
        for (std::uint32_t i = 1; i < n; ++i) {
            const std::uint32_t v = s[i];
            std::uint32_t j = i;
            for (; j > 0 && s[j - 1] > v; --j) s[j] = s[j - 1];
            s[j] = v;
        }
        std::uint32_t out = 0;
        for (std::uint32_t i = 0; i < n;) {
            std::uint32_t j = i + 1;
            while (j < n && s[j] == s[i]) ++j;
            if ((j - i) & 1u) s[out++] = s[i];
            i = j;
        }
        ocnt[t] = out;
    }
}

__global__ void k_odd_write(std::uint64_t n_cp, const std::uint64_t* __restrict__ toff,
                            const std::uint32_t* __restrict__ tbuf, const std::uint32_t* __restrict__ ocnt,
                            const std::uint64_t* __restrict__ ooff, std::uint32_t* __restrict__ top,
                            std::uint32_t* __restrict__ low) {
    AUDIT_STRIDE(t, n_cp) {
        const std::uint64_t o = ooff[t];
        for (std::uint32_t k = 0; k < ocnt[t]; ++k) {
            top[o + k] = static_cast<std::uint32_t>(t);
            low[o + k] = tbuf[toff[t] + k];
        }
    }
}

}  // namespace
}  // namespace msc3d_dev

namespace msc3d_stage {

#define ATRY(x)                          \
    do {                                 \
        const int _rc = (x);             \
        if (_rc != MSC3D_OK) return _rc; \
    } while (0)

int audit_gradient(msc3d_ctx* ctx, std::uint64_t max_cells_for_cycles, std::uint64_t out[4]) {
    using namespace msc3d_dev;
    const auto* codes = ctx->ptr<std::uint8_t>("codes");
    if (!codes) return MSC3D_ERR_STATE;
    const Dims& d = ctx->dims;
    const cudaStream_t s = ctx->stream;
    // [0] violations [1] pairs [2] samples [3] upward-paired; peel counters at 108..112
    auto* stats = reinterpret_cast<unsigned long long*>(ctx->d_small + 96);
    auto* cnt = reinterpret_cast<unsigned long long*>(ctx->d_small + 108);
    auto* samples = static_cast<std::uint64_t*>(ctx->ensure("audit_samples", kSampleCap, 8));
    if (!samples) return MSC3D_ERR_NOMEM;
    MSC3D_CUDA_TRY(cudaMemsetAsync(stats, 0, 4 * 8, s));
    MSC3D_CUDA_TRY(cudaMemsetAsync(cnt, 0, 5 * 8, s));
    k_matching<<<std::min(blocks_for(d.n_cells), 64u * ctx->num_sms), kT, 0, s>>>(codes, d, stats, samples);
    count_launch();
    MSC3D_CUDA_TRY(cudaGetLastError());
    const bool cycles = d.n_cells <= max_cells_for_cycles;
    if (cycles) {
        auto* indeg = static_cast<std::uint32_t*>(ctx->ensure("audit_indeg", d.n_cells, 4));
        auto* fa = static_cast<std::uint64_t*>(ctx->ensure("audit_fa", d.n_cells, 8));
        auto* fb = static_cast<std::uint64_t*>(ctx->ensure("audit_fb", d.n_cells, 8));
        if (!indeg || !fa || !fb) return MSC3D_ERR_NOMEM;
        MSC3D_CUDA_TRY(cudaMemsetAsync(indeg, 0, d.n_cells * 4, s));
        const unsigned g = std::min(blocks_for(d.n_cells), 64u * ctx->num_sms);
        k_vpath_indeg<<<g, kT, 0, s>>>(codes, d, indeg, stats);
        k_vpath_seed<<<g, kT, 0, s>>>(codes, d, indeg, fa, cnt);
        int per_sm = 0;
        MSC3D_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &per_sm, reinterpret_cast<const void*>(k_vpath_peel), kT, 0));
        if (per_sm <= 0) return MSC3D_ERR_CUDA;
        Dims dd = d;
        void* args[] = {&codes, &dd, &indeg, &fa, &fb, &cnt};
        MSC3D_CUDA_TRY(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k_vpath_peel),
                                                   dim3(per_sm * ctx->num_sms), dim3(kT), args, 0, s));
        count_launch(3);
    }
    ATRY(ctx->fetch_range(96, 17));
    const std::uint64_t* h = ctx->h_small + 96;
    out[0] = h[0];                                  // matching_violations
    out[1] = cycles ? h[3] - h[15] : 0;             // cells_in_closed_vpath = upward - peeled
    out[2] = cycles ? 1 : 0;                        // acyclicity_checked
    out[3] = h[1] == 0 ? 1 : 0;                     // degenerate: no pairs at all
    ctx->scalars["audit_samples"] = static_cast<std::int64_t>(std::min<std::uint64_t>(h[2], kSampleCap));
    ctx->scalars["audit_peel_levels"] = static_cast<std::int64_t>(h[16]);
    ctx->find("audit_samples")->count = std::min<std::uint64_t>(h[2], kSampleCap);
    return MSC3D_OK;
}

int boundary_check(msc3d_ctx* ctx, std::uint64_t n_cp, const std::uint8_t* cp_index, std::uint64_t n_arcs,
                   const std::uint32_t* src, const std::uint32_t* dst, const std::uint64_t* mult,
                   std::uint64_t* n_odd) {
    using namespace msc3d_dev;
    const cudaStream_t s = ctx->stream;
    auto* in_cnt = static_cast<std::uint32_t*>(ctx->ensure("bc_in_cnt", std::max<std::uint64_t>(n_cp, 1), 4));
    auto* in_off = static_cast<std::uint64_t*>(ctx->ensure("bc_in_off", std::max<std::uint64_t>(n_cp, 1), 8));
    auto* cursor = static_cast<std::uint32_t*>(ctx->ensure("bc_cursor", std::max<std::uint64_t>(n_cp, 1), 4));
    auto* in_arc = static_cast<std::uint64_t*>(ctx->ensure("bc_in_arc", std::max<std::uint64_t>(n_arcs, 1), 8));
    auto* tcnt = static_cast<std::uint32_t*>(ctx->ensure("bc_tcnt", std::max<std::uint64_t>(n_cp, 1), 4));
    auto* toff = static_cast<std::uint64_t*>(ctx->ensure("bc_toff", std::max<std::uint64_t>(n_cp, 1), 8));
    auto* ocnt = static_cast<std::uint32_t*>(ctx->ensure("bc_ocnt", std::max<std::uint64_t>(n_cp, 1), 4));
    auto* ooff = static_cast<std::uint64_t*>(ctx->ensure("bc_ooff", std::max<std::uint64_t>(n_cp, 1), 8));
    if (!in_cnt || !in_off || !cursor || !in_arc || !tcnt || !toff || !ocnt || !ooff) return MSC3D_ERR_NOMEM;
    *n_odd = 0;
    if (n_cp == 0) {
        ctx->ensure("odd_top", 0, 4);
        ctx->ensure("odd_low", 0, 4);
        return MSC3D_OK;
    }
    auto* flag = reinterpret_cast<unsigned int*>(ctx->d_small + 120);
    MSC3D_CUDA_TRY(cudaMemsetAsync(flag, 0, 8, s));
    MSC3D_CUDA_TRY(cudaMemsetAsync(in_cnt, 0, n_cp * 4, s));
    MSC3D_CUDA_TRY(cudaMemsetAsync(cursor, 0, n_cp * 4, s));
    if (n_arcs) k_in_count<<<blocks_for(n_arcs), kT, 0, s>>>(dst, n_arcs, in_cnt);
    ATRY(scan_u32(in_cnt, n_cp, in_off, ctx->d_small + 121, ctx->ws, s));
    if (n_arcs) k_in_fill<<<blocks_for(n_arcs), kT, 0, s>>>(dst, n_arcs, in_off, cursor, in_arc);
    k_toggles<false><<<blocks_for(n_cp), kT, 0, s>>>(cp_index, n_cp, src, mult, in_off, in_cnt, in_arc, tcnt,
                                                     nullptr, nullptr, flag);
    ATRY(scan_u32(tcnt, n_cp, toff, ctx->d_small + 122, ctx->ws, s));
    ATRY(ctx->fetch_range(120, 3));
    if (static_cast<unsigned int>(ctx->h_small[120])) return MSC3D_ERR_NOMEM;
    const std::uint64_t ntog = ctx->h_small[122];
    auto* tbuf = static_cast<std::uint32_t*>(ctx->ensure("bc_toggles", std::max<std::uint64_t>(ntog, 1), 4));
    if (!tbuf) return MSC3D_ERR_NOMEM;
    k_toggles<true><<<blocks_for(n_cp), kT, 0, s>>>(cp_index, n_cp, src, mult, in_off, in_cnt, in_arc, tcnt, toff,
                                                    tbuf, flag);
    k_toggle_parity<<<blocks_for(n_cp), kT, 0, s>>>(n_cp, toff, tcnt, tbuf, ocnt);
    ATRY(scan_u32(ocnt, n_cp, ooff, ctx->d_small + 123, ctx->ws, s));
    ATRY(ctx->fetch_range(123, 1));
    const std::uint64_t nodd = ctx->h_small[123];
    auto* top = static_cast<std::uint32_t*>(ctx->ensure("odd_top", nodd, 4));
    auto* low = static_cast<std::uint32_t*>(ctx->ensure("odd_low", nodd, 4));
    if (!top || !low) return MSC3D_ERR_NOMEM;
    if (nodd) k_odd_write<<<blocks_for(n_cp), kT, 0, s>>>(n_cp, toff, tbuf, ocnt, ooff, top, low);
    count_launch(nodd ? 6 : 5);
    MSC3D_CUDA_TRY(cudaGetLastError());
    MSC3D_CUDA_TRY(cudaStreamSynchronize(s));
    *n_odd = nodd;
    return MSC3D_OK;
}

}  // namespace msc3d_stage

// Critical-cell extraction (extract_critical_cells, proj/src/gradient.cpp:285-297):
// one pass over the N pair codes, four ascending id lists (one per dimension).
//
// Each thread reads 16 consecutive codes with one 16-byte load (vectorised,
// coalesced), derives each cell's dimension from its lattice coordinates (one
// 64-bit division per 16 cells, then incremental), and counts critical cells per
// dimension.  Counts are packed 16 bits per dimension, block-scanned with warp
// shuffles, and chained across tiles by decoupled look-back (scan.cuh); the ids
// are then written in ascending order.  The same kernel family also serves every
// other "cells of dimension d satisfying P, ascending" compaction of the
// reference (stream_compact_indices, primitives.hpp:147-182) through the Pred
// functor.
#include <algorithm>

#include "common.cuh"
#include "kernels.cuh"
#include "scan.cuh"

namespace msc3d_dev {

namespace {

constexpr int kThreads = 256;
constexpr int kChunks = 4;                  // 16-byte loads per thread
constexpr int kPerThread = 16 * kChunks;    // codes per thread
constexpr int kTile = kThreads * kPerThread;  // 16384 codes: per-category tile counts < 2^16

// A predicate maps (cell id, code, dimension) to an output list (0..3) or -1.
struct CritPred {
    __device__ __forceinline__ int operator()(std::uint64_t, std::uint8_t code, int dm) const {
        return code == kCritical ? dm : -1;
    }
};

// Marked critical cells (mark_reachable's one_saddles / two_saddles compaction,
// saddle_graph.cpp:71-85).
struct MarkedCritPred {
    const std::uint8_t* marked;
    __device__ __forceinline__ int operator()(std::uint64_t i, std::uint8_t code, int dm) const {
        return (code == kCritical && marked[i]) ? dm : -1;
    }
};

// All critical saddles (dims 1 and 2) into ONE ascending list: the merged saddle
// order of saddle_extremum_arcs (extrema.cpp:109-117).
struct SaddlePred {
    __device__ __forceinline__ int operator()(std::uint64_t, std::uint8_t code, int dm) const {
        return (code == kCritical && (dm == 1 || dm == 2)) ? 0 : -1;
    }
};

// Junctions of a marked subgraph (saddle_graph.cpp:126-133), ascending.
struct JunctionPred {
    const std::uint8_t* codes;
    const std::uint8_t* marked;
    Dims d;
    __device__ __forceinline__ int operator()(std::uint64_t i, std::uint8_t code, int dm) const {
        if (dm != 1 || code == kCritical || !marked[i]) return -1;
        const Coord c = unpack(d, i);
        return edge_successor_count(codes, d, c.x, c.y, c.z) > 1 ? 0 : -1;
    }
};

template <typename Pred, typename IdT>
__global__ void __launch_bounds__(kThreads)
k_compact_by_dim(const std::uint8_t* __restrict__ codes, Dims d, Pred pred, TileStatus st,
                 IdT* out0, IdT* out1, IdT* out2, IdT* out3, std::uint64_t* totals) {
    __shared__ std::uint64_t sm[40];
    __shared__ std::uint32_t s_tile;
    if (threadIdx.x == 0) s_tile = atomicAdd(st.ticket, 1u);
    __syncthreads();
    const std::uint32_t tile = s_tile;
    const std::uint64_t first = static_cast<std::uint64_t>(tile) * kTile +
                                static_cast<std::uint64_t>(threadIdx.x) * kPerThread;

    // kPerThread codes: kChunks 16-byte loads issued back to back
    std::uint32_t ws[kPerThread / 4];
    if (first + kPerThread <= d.n_cells && (first & 15) == 0) {
#pragma unroll
        for (int q = 0; q < kChunks; ++q) {
            const uint4 w = *reinterpret_cast<const uint4*>(codes + first + 16 * q);
            ws[4 * q] = w.x;
            ws[4 * q + 1] = w.y;
            ws[4 * q + 2] = w.z;
            ws[4 * q + 3] = w.w;
        }
    } else {
#pragma unroll
        for (int q = 0; q < kPerThread / 4; ++q) {
            std::uint32_t v = 0;
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const std::uint64_t i = first + 4 * q + b;
                v |= static_cast<std::uint32_t>(i < d.n_cells ? codes[i] : kUnset) << (8 * b);
            }
            ws[q] = v;
        }
    }

    // Lattice coordinates of the first cell; dims of the following ones by
    // incrementing x with carries.
    Coord p = unpack(d, first < d.n_cells ? first : 0);
    std::uint32_t dimbits[kChunks];  // 2 bits per cell: output list
    std::uint32_t hit[kChunks];      // 1 bit per cell: predicate
    std::uint64_t packed = 0;
#pragma unroll
    for (int q = 0; q < kChunks; ++q) {
        dimbits[q] = 0;
        hit[q] = 0;
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            const std::uint8_t c = static_cast<std::uint8_t>(ws[(16 * q + k) >> 2] >> (8 * (k & 3)));
            const std::uint64_t i = first + 16 * q + k;
            const int dm0 = static_cast<int>((p.x & 1) + (p.y & 1) + (p.z & 1));
            const int dm = i < d.n_cells ? pred(i, c, dm0) : -1;
            if (dm >= 0) {
                dimbits[q] |= static_cast<std::uint32_t>(dm) << (2 * k);
                hit[q] |= 1u << k;
                packed += 1ull << (16 * dm);
            }
            if (++p.x == d.ex) {
                p.x = 0;
                if (++p.y == d.ey) {
                    p.y = 0;
                    ++p.z;
                }
            }
        }
    }

    std::uint64_t block_total;
    const std::uint64_t excl = block_excl_scan(packed, &block_total, sm);
    std::uint64_t tot[4];
    for (int k = 0; k < 4; ++k) tot[k] = unpack16(block_total, k);
    tile_lookback4(st, tile, tot, sm + 34);

    std::uint64_t at[4];
    for (int k = 0; k < 4; ++k) at[k] = sm[34 + k] + unpack16(excl, k);
    IdT* outs[4] = {out0, out1, out2, out3};
#pragma unroll
    for (int q = 0; q < kChunks; ++q)
        for (std::uint32_t m = hit[q]; m; m &= m - 1) {
            const int k = __ffs(m) - 1;
            const int dm = (dimbits[q] >> (2 * k)) & 3;
            if (outs[dm]) outs[dm][at[dm]] = static_cast<IdT>(first + 16 * q + k);
            ++at[dm];
        }
    const std::uint32_t ntiles = static_cast<std::uint32_t>((d.n_cells + kTile - 1) / kTile);
    if (tile == ntiles - 1 && threadIdx.x == 0 && totals) {
        for (int k = 0; k < 4; ++k) totals[k] = sm[34 + k] + tot[k];
    }
}

// The critical-cell compaction proper (CritPred), bit-parallel: a thread's 64 codes
// become a 64-bit "critical" mask (byte compares, __vcmpeq4); within one lattice row
// the cell dimension is (row parity) + (x parity), so the four per-dimension masks
// are the critical mask ANDed with alternating-bit masks of the (at most two, since
// ex >= 64) rows the thread spans.  Counts are popcounts; ids are written by walking
// the set bits.  ~10x fewer instructions than the per-cell loop above.
template <typename IdT>
__global__ void __launch_bounds__(kThreads)
k_compact_crit(const std::uint8_t* __restrict__ codes, Dims d, TileStatus st, IdT* out0, IdT* out1, IdT* out2,
               IdT* out3, std::uint64_t* totals) {
    static_assert(kPerThread == 64, "one 64-bit mask per thread");
    __shared__ std::uint64_t sm[40];
    __shared__ std::uint32_t s_tile;
    if (threadIdx.x == 0) s_tile = atomicAdd(st.ticket, 1u);
    __syncthreads();
    const std::uint32_t tile = s_tile;
    const std::uint64_t first = static_cast<std::uint64_t>(tile) * kTile +
                                static_cast<std::uint64_t>(threadIdx.x) * kPerThread;
    std::uint64_t crit = 0;
    if (first + kPerThread <= d.n_cells) {
#pragma unroll
        for (int q = 0; q < kChunks; ++q) {
            const uint4 w = *reinterpret_cast<const uint4*>(codes + first + 16 * q);
            const std::uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const std::uint32_t m = __vcmpeq4(ws[e], 0x01010101u);  // kCritical bytes -> 0xff
                const std::uint64_t b4 = ((m >> 7) & 1u) | ((m >> 14) & 2u) | ((m >> 21) & 4u) | ((m >> 28) & 8u);
                crit |= b4 << (16 * q + 4 * e);
            }
        }
    } else {
        for (int k = 0; k < kPerThread; ++k)
            if (first + k < d.n_cells && codes[first + k] == kCritical) crit |= 1ull << k;
    }
    // rows spanned: A = cells [0, lenA), B = the rest
    const Coord p = unpack(d, first < d.n_cells ? first : 0);
    const std::uint64_t lenA = min(static_cast<std::uint64_t>(kPerThread), static_cast<std::uint64_t>(d.ex - p.x));
    const std::uint64_t segA = lenA >= 64 ? ~0ull : ((1ull << lenA) - 1);
    constexpr std::uint64_t kAlt = 0xAAAAAAAAAAAAAAAAull;  // odd k
    const std::uint64_t oddA = (p.x & 1) ? ~kAlt : kAlt;   // cells of row A with odd x
    const std::uint64_t oddB = (lenA & 1) ? ~kAlt : kAlt;
    std::int64_t yB = p.y + 1, zB = p.z;
    if (yB == d.ey) {
        yB = 0;
        ++zB;
    }
    const int rA = static_cast<int>((p.y & 1) + (p.z & 1));
    const int rB = static_cast<int>((yB & 1) + (zB & 1));
    const std::uint64_t cA = crit & segA, cB = crit & ~segA;
    std::uint64_t M[4];
#pragma unroll
    for (int dm = 0; dm < 4; ++dm)
        M[dm] = (rA == dm ? (cA & ~oddA) : 0ull) | (rA + 1 == dm ? (cA & oddA) : 0ull) |
                (rB == dm ? (cB & ~oddB) : 0ull) | (rB + 1 == dm ? (cB & oddB) : 0ull);
    std::uint64_t packed = 0;
#pragma unroll
    for (int dm = 0; dm < 4; ++dm) packed += static_cast<std::uint64_t>(__popcll(M[dm])) << (16 * dm);

    std::uint64_t block_total;
    const std::uint64_t excl = block_excl_scan(packed, &block_total, sm);
    std::uint64_t tot[4];
    for (int k = 0; k < 4; ++k) tot[k] = unpack16(block_total, k);
    tile_lookback4(st, tile, tot, sm + 34);
    IdT* outs[4] = {out0, out1, out2, out3};
#pragma unroll
    for (int dm = 0; dm < 4; ++dm) {
        std::uint64_t at = sm[34 + dm] + unpack16(excl, dm);
        for (std::uint64_t m = M[dm]; m; m &= m - 1) outs[dm][at++] = static_cast<IdT>(first + __ffsll(m) - 1);
    }
    const std::uint32_t ntiles = static_cast<std::uint32_t>((d.n_cells + kTile - 1) / kTile);
    if (tile == ntiles - 1 && threadIdx.x == 0 && totals) {
        for (int k = 0; k < 4; ++k) totals[k] = sm[34 + k] + tot[k];
    }
}

// Per-dimension masks of the critical cells among the 64 cells [first, first + 64)
// (bit k = cell first + k): byte compares to bits, then lattice parity masks.
// Critical-code bits of 64 consecutive cells, from four 16-byte words.
__device__ __forceinline__ std::uint64_t crit_bits(const uint4 (&w4)[kChunks]) {
    std::uint64_t crit = 0;
#pragma unroll
    for (int q = 0; q < kChunks; ++q) {
        const std::uint32_t ws[4] = {w4[q].x, w4[q].y, w4[q].z, w4[q].w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const std::uint32_t m = __vcmpeq4(ws[e], 0x01010101u);  // kCritical bytes -> 0xff
            const std::uint64_t b4 = ((m >> 7) & 1u) | ((m >> 14) & 2u) | ((m >> 21) & 4u) | ((m >> 28) & 8u);
            crit |= b4 << (16 * q + 4 * e);
        }
    }
    return crit;
}

// Per-dimension masks of the 64 cells starting at `first` from their critical bits.
__device__ __forceinline__ void crit_dim_masks(std::uint64_t crit, const Dims& d, std::uint64_t first,
                                               std::uint64_t M[4]);

__device__ __forceinline__ void crit_chunk_masks(const std::uint8_t* __restrict__ codes, const Dims& d,
                                                 std::uint64_t first, std::uint64_t M[4]) {
    std::uint64_t crit = 0;
    if (first + kPerThread <= d.n_cells) {
#pragma unroll
        for (int q = 0; q < kChunks; ++q) {
            const uint4 w = __ldcs(reinterpret_cast<const uint4*>(codes + first + 16 * q));
            const std::uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const std::uint32_t m = __vcmpeq4(ws[e], 0x01010101u);  // kCritical bytes -> 0xff
                const std::uint64_t b4 = ((m >> 7) & 1u) | ((m >> 14) & 2u) | ((m >> 21) & 4u) | ((m >> 28) & 8u);
                crit |= b4 << (16 * q + 4 * e);
            }
        }
    } else {
        for (int k = 0; k < kPerThread; ++k)
            if (first + k < d.n_cells && codes[first + k] == kCritical) crit |= 1ull << k;
    }
    crit_dim_masks(crit, d, first, M);
}

__device__ __forceinline__ void crit_dim_masks(std::uint64_t crit, const Dims& d, std::uint64_t first,
                                               std::uint64_t M[4]) {
    const Coord p = unpack(d, first < d.n_cells ? first : 0);
    const std::uint64_t lenA = min(static_cast<std::uint64_t>(kPerThread), static_cast<std::uint64_t>(d.ex - p.x));
    const std::uint64_t segA = lenA >= 64 ? ~0ull : ((1ull << lenA) - 1);
    constexpr std::uint64_t kAlt = 0xAAAAAAAAAAAAAAAAull;  // odd k
    const std::uint64_t oddA = (p.x & 1) ? ~kAlt : kAlt;
    const std::uint64_t oddB = (lenA & 1) ? ~kAlt : kAlt;
    std::int64_t yB = p.y + 1, zB = p.z;
    if (yB == d.ey) {
        yB = 0;
        ++zB;
    }
    const int rA = static_cast<int>((p.y & 1) + (p.z & 1));
    const int rB = static_cast<int>((yB & 1) + (zB & 1));
    const std::uint64_t cA = crit & segA, cB = crit & ~segA;
#pragma unroll
    for (int dm = 0; dm < 4; ++dm)
        M[dm] = (rA == dm ? (cA & ~oddA) : 0ull) | (rA + 1 == dm ? (cA & oddA) : 0ull) |
                (rB == dm ? (cB & ~oddB) : 0ull) | (rB + 1 == dm ? (cB & oddB) : 0ull);
}

// Counts only (when the gradient kernel's totals are not available, e.g. codes
// installed from outside): the same masks, block reduction, one atomic per block
// and dimension.
#define CRIT_GRID_STRIDE(i, n)                                                                  \
    for (std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x; i < (n); \
         i += static_cast<std::uint64_t>(gridDim.x) * blockDim.x)
__global__ void __launch_bounds__(kThreads)
k_count_crit(const std::uint8_t* __restrict__ codes, Dims d, unsigned long long* __restrict__ totals) {
    __shared__ unsigned long long s[4];
    if (threadIdx.x < 4) s[threadIdx.x] = 0;
    __syncthreads();
    unsigned long long local[4] = {0, 0, 0, 0};
    const std::uint64_t nchunks = (d.n_cells + kPerThread - 1) / kPerThread;
    CRIT_GRID_STRIDE(c, nchunks) {
        std::uint64_t M[4];
        crit_chunk_masks(codes, d, c * kPerThread, M);
#pragma unroll
        for (int dm = 0; dm < 4; ++dm) local[dm] += __popcll(M[dm]);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        unsigned long long v = local[k];
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if ((threadIdx.x & 31) == 0 && v) atomicAdd(&s[k], v);
    }
    __syncthreads();
    if (threadIdx.x < 4 && s[threadIdx.x]) atomicAdd(&totals[threadIdx.x], s[threadIdx.x]);
}

// Three 64-cell chunks per thread (49152-cell tiles: per-category tile counts still fit
// 16 bits; a thread's chunks are consecutive, so thread order is cell order) amortise
// the look-back; the tile's ids are staged in shared memory and
// leave as contiguous runs per category (coalesced), unless the tile holds more than
// kStage of them (then direct per-thread writes, as in k_compact_crit).
constexpr int kSub = 3;
constexpr int kStageBytes = 32768;
template <typename IdT>
__global__ void __launch_bounds__(kThreads)
k_compact_crit3(const std::uint8_t* __restrict__ codes, Dims d, TileStatus st, IdT* out0, IdT* out1, IdT* out2,
                IdT* out3, std::uint64_t* totals) {
    static_assert(kPerThread == 64, "one 64-bit mask per thread and sub-tile");
    __shared__ std::uint64_t sm[40];
    __shared__ std::uint32_t s_tile;
    constexpr int kStage = kStageBytes / static_cast<int>(sizeof(IdT));
    __shared__ IdT s_ids[kStage];
    if (threadIdx.x == 0) s_tile = atomicAdd(st.ticket, 1u);
    __syncthreads();
    const std::uint32_t tile = s_tile;
    std::uint64_t M[kSub][4];
    std::uint64_t packed = 0;
    const std::uint64_t first0 = static_cast<std::uint64_t>(tile) * kSub * kTile +
                                 static_cast<std::uint64_t>(threadIdx.x) * kSub * kPerThread;
    if (static_cast<std::uint64_t>(tile + 1) * kSub * kTile <= d.n_cells) {
        // a full tile: the thread's twelve 16-byte loads issued back to back, then the masks
        uint4 w4[kSub][kChunks];
        const uint4* src = reinterpret_cast<const uint4*>(codes + first0);
#pragma unroll
        for (int sb = 0; sb < kSub; ++sb)
#pragma unroll
            for (int q = 0; q < kChunks; ++q) w4[sb][q] = __ldcs(src + sb * kChunks + q);
#pragma unroll
        for (int sb = 0; sb < kSub; ++sb) crit_dim_masks(crit_bits(w4[sb]), d, first0 + sb * kPerThread, M[sb]);
    } else {
#pragma unroll
        for (int sb = 0; sb < kSub; ++sb) crit_chunk_masks(codes, d, first0 + sb * kPerThread, M[sb]);
    }
#pragma unroll
    for (int sb = 0; sb < kSub; ++sb)
#pragma unroll
        for (int dm = 0; dm < 4; ++dm) packed += static_cast<std::uint64_t>(__popcll(M[sb][dm])) << (16 * dm);
    std::uint64_t block_total;
    const std::uint64_t excl = block_excl_scan(packed, &block_total, sm);
    std::uint64_t tot[4];
    for (int k = 0; k < 4; ++k) tot[k] = unpack16(block_total, k);
    tile_lookback4(st, tile, tot, sm + 34);
    IdT* outs[4] = {out0, out1, out2, out3};
    const std::uint64_t ttot = tot[0] + tot[1] + tot[2] + tot[3];
    if (ttot <= static_cast<std::uint64_t>(kStage)) {
        // tile-local positions: categories one after another
        std::uint64_t cbase = 0;
#pragma unroll
        for (int dm = 0; dm < 4; ++dm) {
            std::uint64_t at = cbase + unpack16(excl, dm);
#pragma unroll
            for (int sb = 0; sb < kSub; ++sb) {
                const std::uint64_t first = static_cast<std::uint64_t>(tile) * kSub * kTile +
                                            (static_cast<std::uint64_t>(threadIdx.x) * kSub + sb) * kPerThread;
                for (std::uint64_t m = M[sb][dm]; m; m &= m - 1)
                    s_ids[at++] = static_cast<IdT>(first + __ffsll(m) - 1);
            }
            cbase += tot[dm];
        }
        __syncthreads();
        cbase = 0;
#pragma unroll
        for (int dm = 0; dm < 4; ++dm) {
            IdT* dst = outs[dm] + sm[34 + dm];
            for (std::uint64_t j = threadIdx.x; j < tot[dm]; j += kThreads) dst[j] = s_ids[cbase + j];
            cbase += tot[dm];
        }
    } else {
#pragma unroll
        for (int dm = 0; dm < 4; ++dm) {
            std::uint64_t at = sm[34 + dm] + unpack16(excl, dm);
#pragma unroll
            for (int sb = 0; sb < kSub; ++sb) {
                const std::uint64_t first = static_cast<std::uint64_t>(tile) * kSub * kTile +
                                            (static_cast<std::uint64_t>(threadIdx.x) * kSub + sb) * kPerThread;
                for (std::uint64_t m = M[sb][dm]; m; m &= m - 1)
                    outs[dm][at++] = static_cast<IdT>(first + __ffsll(m) - 1);
            }
        }
    }
    const std::uint32_t ntiles = static_cast<std::uint32_t>((d.n_cells + kSub * kTile - 1) / (kSub * kTile));
    if (tile == ntiles - 1 && threadIdx.x == 0 && totals) {
        for (int k = 0; k < 4; ++k) totals[k] = sm[34 + k] + tot[k];
    }
}

// Count-only pass: totals per dimension with block reduction + one atomic per block.
template <typename Pred>
__global__ void __launch_bounds__(kThreads)
k_count_by_dim(const std::uint8_t* __restrict__ codes, Dims d, Pred pred,
               unsigned long long* totals) {
    __shared__ unsigned long long s[4];
    if (threadIdx.x < 4) s[threadIdx.x] = 0;
    __syncthreads();
    unsigned long long local[4] = {0, 0, 0, 0};
    const std::uint64_t stride = static_cast<std::uint64_t>(gridDim.x) * kTile;
    for (std::uint64_t tbase = static_cast<std::uint64_t>(blockIdx.x) * kTile; tbase < d.n_cells;
         tbase += stride) {
        const std::uint64_t first = tbase + static_cast<std::uint64_t>(threadIdx.x) * kPerThread;
        if (first >= d.n_cells) continue;
        Coord p = unpack(d, first);
        for (int k = 0; k < kPerThread && first + k < d.n_cells; ++k) {
            const std::uint8_t c = codes[first + k];
            const int cat = pred(first + k, c, static_cast<int>((p.x & 1) + (p.y & 1) + (p.z & 1)));
            if (cat >= 0) ++local[cat];
            if (++p.x == d.ex) {
                p.x = 0;
                if (++p.y == d.ey) {
                    p.y = 0;
                    ++p.z;
                }
            }
        }
    }
    for (int k = 0; k < 4; ++k) {
        unsigned long long v = local[k];
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if ((threadIdx.x & 31) == 0 && v) atomicAdd(&s[k], v);
    }
    __syncthreads();
    if (threadIdx.x < 4 && s[threadIdx.x]) atomicAdd(&totals[threadIdx.x], s[threadIdx.x]);
}

template <typename Pred>
int compact_impl(const std::uint8_t* codes, const Dims& d, Pred pred, Workspace& ws,
                 void* const outs[4], int id_width, std::uint64_t* d_totals, cudaStream_t s) {
    const std::uint64_t ntiles = (d.n_cells + kTile - 1) / kTile;
    if (ntiles == 0) return MSC3D_OK;
    if (ntiles > 0xffffffffull) return MSC3D_ERR_INVALID;
    TileStatus st;
    const std::size_t bytes = ntiles * (4 + 64) + 16;
    char* buf = static_cast<char*>(ws.get(bytes));
    if (!buf) return MSC3D_ERR_NOMEM;
    st.agg = reinterpret_cast<std::uint64_t*>(buf);
    st.incl = st.agg + 4 * ntiles;
    st.flag = reinterpret_cast<std::uint32_t*>(st.incl + 4 * ntiles);
    st.ticket = st.flag + ntiles;
    MSC3D_CUDA_TRY(cudaMemsetAsync(st.flag, 0, (ntiles + 1) * 4, s));
    const dim3 grid(static_cast<unsigned>(ntiles));
    if (id_width == 4)
        k_compact_by_dim<Pred, std::uint32_t><<<grid, kThreads, 0, s>>>(
            codes, d, pred, st, static_cast<std::uint32_t*>(outs[0]),
            static_cast<std::uint32_t*>(outs[1]), static_cast<std::uint32_t*>(outs[2]),
            static_cast<std::uint32_t*>(outs[3]), d_totals);
    else
        k_compact_by_dim<Pred, std::uint64_t><<<grid, kThreads, 0, s>>>(
            codes, d, pred, st, static_cast<std::uint64_t*>(outs[0]),
            static_cast<std::uint64_t*>(outs[1]), static_cast<std::uint64_t*>(outs[2]),
            static_cast<std::uint64_t*>(outs[3]), d_totals);
    count_launch();
    MSC3D_CUDA_TRY(cudaGetLastError());
    return MSC3D_OK;
}

template <typename Pred>
int count_impl(const std::uint8_t* codes, const Dims& d, Pred pred, std::uint64_t* d_totals,
               cudaStream_t s, int num_sms) {
    MSC3D_CUDA_TRY(cudaMemsetAsync(d_totals, 0, 32, s));
    const std::uint64_t ntiles = (d.n_cells + kTile - 1) / kTile;
    const unsigned grid = static_cast<unsigned>(std::min<std::uint64_t>(ntiles, 8ull * num_sms));
    k_count_by_dim<Pred><<<grid, kThreads, 0, s>>>(codes, d, pred,
                                                   reinterpret_cast<unsigned long long*>(d_totals));
    count_launch();
    MSC3D_CUDA_TRY(cudaGetLastError());
    return MSC3D_OK;
}

}  // namespace

int launch_critical_count(const std::uint8_t* codes, const Dims& d, std::uint64_t* d_totals,
                          cudaStream_t s, int num_sms) {
    if (d.ex < 64) return count_impl(codes, d, CritPred{}, d_totals, s, num_sms);
    MSC3D_CUDA_TRY(cudaMemsetAsync(d_totals, 0, 32, s));
    const std::uint64_t nchunks = (d.n_cells + kPerThread - 1) / kPerThread;
    const unsigned grid = static_cast<unsigned>(std::min<std::uint64_t>((nchunks + kThreads - 1) / kThreads,
                                                                        static_cast<std::uint64_t>(num_sms) * 16));
    k_count_crit<<<grid, kThreads, 0, s>>>(codes, d, reinterpret_cast<unsigned long long*>(d_totals));
    count_launch();
    MSC3D_CUDA_TRY(cudaGetLastError());
    return MSC3D_OK;
}

int launch_critical_compact(const std::uint8_t* codes, const Dims& d, Workspace& ws,
                            void* const outs[4], int id_width, std::uint64_t* d_totals,
                            cudaStream_t s) {
    if (d.ex < 64 || !outs[0] || !outs[1] || !outs[2] || !outs[3] || d.n_cells == 0)
        return compact_impl(codes, d, CritPred{}, ws, outs, id_width, d_totals, s);
    const std::uint64_t ntiles = (d.n_cells + kSub * kTile - 1) / (kSub * kTile);
    char* buf = static_cast<char*>(ws.get(ntiles * 68 + 16));
    if (!buf) return MSC3D_ERR_NOMEM;
    TileStatus st;
    st.agg = reinterpret_cast<std::uint64_t*>(buf);
    st.incl = st.agg + 4 * ntiles;
    st.flag = reinterpret_cast<std::uint32_t*>(st.incl + 4 * ntiles);
    st.ticket = st.flag + ntiles;
    MSC3D_CUDA_TRY(cudaMemsetAsync(st.flag, 0, (ntiles + 1) * 4, s));
    if (id_width == 4)
        k_compact_crit3<std::uint32_t><<<static_cast<unsigned>(ntiles), kThreads, 0, s>>>(
            codes, d, st, static_cast<std::uint32_t*>(outs[0]), static_cast<std::uint32_t*>(outs[1]),
            static_cast<std::uint32_t*>(outs[2]), static_cast<std::uint32_t*>(outs[3]), d_totals);
    else
        k_compact_crit3<std::uint64_t><<<static_cast<unsigned>(ntiles), kThreads, 0, s>>>(
            codes, d, st, static_cast<std::uint64_t*>(outs[0]), static_cast<std::uint64_t*>(outs[1]),
            static_cast<std::uint64_t*>(outs[2]), static_cast<std::uint64_t*>(outs[3]), d_totals);
    count_launch();
    MSC3D_CUDA_TRY(cudaGetLastError());
    return MSC3D_OK;
}

int launch_saddle_count(const std::uint8_t* codes, const Dims& d, std::uint64_t* d_totals,
                        cudaStream_t s, int num_sms) {
    return count_impl(codes, d, SaddlePred{}, d_totals, s, num_sms);
}

int launch_saddle_compact(const std::uint8_t* codes, const Dims& d, Workspace& ws, void* out,
                          int id_width, std::uint64_t* d_totals, cudaStream_t s) {
    void* const outs[4] = {out, nullptr, nullptr, nullptr};
    return compact_impl(codes, d, SaddlePred{}, ws, outs, id_width, d_totals, s);
}

int launch_junction_cells(const std::uint8_t* codes, const std::uint8_t* marked, const Dims& d,
                          Workspace& ws, void* out, int id_width, std::uint64_t* d_totals,
                          cudaStream_t s, int num_sms, bool count_only) {
    const JunctionPred pred{codes, marked, d};
    if (count_only) return count_impl(codes, d, pred, d_totals, s, num_sms);
    void* const outs[4] = {out, nullptr, nullptr, nullptr};
    return compact_impl(codes, d, pred, ws, outs, id_width, d_totals, s);
}

int launch_marked_critical_count(const std::uint8_t* codes, const std::uint8_t* marked,
                                 const Dims& d, std::uint64_t* d_totals, cudaStream_t s,
                                 int num_sms) {
    return count_impl(codes, d, MarkedCritPred{marked}, d_totals, s, num_sms);
}

int launch_marked_critical_compact(const std::uint8_t* codes, const std::uint8_t* marked,
                                   const Dims& d, Workspace& ws, void* const outs[4],
                                   int id_width, std::uint64_t* d_totals, cudaStream_t s) {
    return compact_impl(codes, d, MarkedCritPred{marked}, ws, outs, id_width, d_totals, s);
}

}  // namespace msc3d_dev

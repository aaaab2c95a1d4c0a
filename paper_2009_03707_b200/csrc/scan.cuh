// Single-pass prefix scan with decoupled look-back (Merrill & Garland), hand-written:
// no CUB/Thrust.  Replaces the reference's chunked two-pass prefix_sum /
// stream_compact(_indices) (proj/include/msc3d/primitives.hpp:48-182).
//
// A "tile" publishes FOUR 64-bit running counts at once (one per cell dimension /
// category), so one pass over the codes compacts all four critical lists
// (gradient.cpp:285-297 runs four separate passes).  Within a tile, the per-thread
// counts are packed 16 bits per category into one u64 and block-scanned with warp
// shuffles; tile totals must stay < 65536 per category.
#pragma once

#include <cstdint>

#include "common.cuh"

namespace msc3d_dev {

struct TileStatus {
    // flag: 0 = nothing, 1 = aggregate published, 2 = inclusive prefix published.
    std::uint32_t* flag;
    std::uint64_t* agg;   // [tile][4]
    std::uint64_t* incl;  // [tile][4]
    std::uint32_t* ticket;  // dynamic tile id counter (tiles must be claimed in order)
};

__device__ __forceinline__ std::uint64_t unpack16(std::uint64_t p, int k) {
    return (p >> (16 * k)) & 0xffffu;
}

// Inclusive warp scan of a packed u64.
__device__ __forceinline__ std::uint64_t warp_incl_scan(std::uint64_t v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const std::uint64_t n = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += n;
    }
    return v;
}

// Block-wide exclusive scan of a packed u64 (blockDim.x threads, 1-D block, <= 1024).
// Returns this thread's exclusive prefix; *total receives the block total.
__device__ __forceinline__ std::uint64_t block_excl_scan(std::uint64_t v, std::uint64_t* total,
                                                         std::uint64_t* smem /* >= 33 */) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nwarps = (blockDim.x + 31) >> 5;
    const std::uint64_t inc = warp_incl_scan(v);
    if (lane == 31) smem[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        std::uint64_t w = lane < nwarps ? smem[lane] : 0;
        w = warp_incl_scan(w);
        if (lane < nwarps) smem[lane] = w;  // inclusive per warp
        if (lane == nwarps - 1) smem[32] = w;
    }
    __syncthreads();
    const std::uint64_t warp_base = warp > 0 ? smem[warp - 1] : 0;
    *total = smem[32];
    const std::uint64_t r = warp_base + inc - v;
    __syncthreads();
    return r;
}

__device__ __forceinline__ std::uint32_t ld_acquire(const std::uint32_t* p) {
    std::uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(std::uint32_t* p, std::uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Called by ALL threads of the block after the block total (4 categories,
// unpacked) is known.  Returns the 4 exclusive prefixes of this tile in out[4]
// (valid in every thread).  `smem4` must hold >= 4 u64.
__device__ __forceinline__ void tile_lookback4(const TileStatus st, std::uint32_t tile,
                                               const std::uint64_t tot[4], std::uint64_t* smem4) {
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        if (lane == 0) {
            for (int k = 0; k < 4; ++k) {
                st.agg[4ull * tile + k] = tot[k];
                if (tile == 0) st.incl[k] = tot[k];
            }
            st_release(&st.flag[tile], tile == 0 ? 2u : 1u);
        }
        std::uint64_t excl[4] = {0, 0, 0, 0};
        if (tile > 0) {
            std::int64_t pred = static_cast<std::int64_t>(tile) - 1;
            for (;;) {
                const std::int64_t idx = pred - lane;
                std::uint32_t fl = 2;
                std::uint64_t v[4] = {0, 0, 0, 0};
                if (idx >= 0) {
                    do {
                        fl = ld_acquire(&st.flag[idx]);
                    } while (fl == 0);
                    const std::uint64_t* src = fl == 2 ? &st.incl[4 * idx] : &st.agg[4 * idx];
                    for (int k = 0; k < 4; ++k)
                        v[k] = *reinterpret_cast<const volatile std::uint64_t*>(src + k);
                }
                const std::uint32_t incl_mask = __ballot_sync(0xffffffffu, fl == 2);
                // lanes up to (and including) the first inclusive one contribute
                const int stop = incl_mask ? __ffs(incl_mask) - 1 : 31;
                for (int k = 0; k < 4; ++k) {
                    std::uint64_t x = lane <= stop ? v[k] : 0;
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
                    excl[k] += x;
                }
                if (incl_mask) break;
                pred -= 32;
            }
            if (lane == 0) {
                for (int k = 0; k < 4; ++k) st.incl[4ull * tile + k] = excl[k] + tot[k];
                st_release(&st.flag[tile], 2u);
            }
        }
        if (lane == 0)
            for (int k = 0; k < 4; ++k) smem4[k] = excl[k];
    }
    __syncthreads();
}

}  // namespace msc3d_dev

// Device-wide data-parallel primitives (the reference's primitives.hpp, re-designed):
//   * exclusive prefix sum of u32 counts -> u64 offsets, single pass, decoupled
//     look-back (prefix_sum, primitives.hpp:48-106);
//   * gather / iota helpers used by the stage code.
// Hand-written; no CUB/Thrust.
#include <algorithm>

#include "common.cuh"
#include "kernels.cuh"
#include "scan.cuh"

namespace msc3d_dev {

namespace {

constexpr int kThreads = 256;
constexpr int kItems = 16;
constexpr int kTile = kThreads * kItems;

// Single-value decoupled look-back over packed status words: bits 62-63 = 0 none,
// 1 aggregate, 2 inclusive prefix; bits 0-61 = the value (one 8-byte load per
// predecessor).  Called by all threads; returns the tile's exclusive prefix.
__device__ __forceinline__ std::uint64_t tile_lookback1(unsigned long long* status, std::uint32_t tile,
                                                        std::uint64_t tot, std::uint64_t* smem1) {
    constexpr unsigned long long kAgg = 1ull << 62, kIncl = 2ull << 62, kVal = (1ull << 62) - 1;
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        if (lane == 0)
            asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(status + tile),
                         "l"((tile == 0 ? kIncl : kAgg) | tot) : "memory");
        std::uint64_t excl = 0;
        if (tile > 0) {
            std::int64_t pred = static_cast<std::int64_t>(tile) - 1;
            for (;;) {
                const std::int64_t idx = pred - lane;
                unsigned long long w = kIncl;  // (before tile 0: an empty inclusive prefix)
                if (idx >= 0) {
                    do {
                        asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(w) : "l"(status + idx) : "memory");
                    } while ((w >> 62) == 0);
                }
                const std::uint32_t incl_mask = __ballot_sync(0xffffffffu, (w >> 62) == 2);
                const int stop = incl_mask ? __ffs(incl_mask) - 1 : 31;
                std::uint64_t x = lane <= stop ? (w & kVal) : 0;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
                excl += x;
                if (incl_mask) break;
                pred -= 32;
            }
            if (lane == 0)
                asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(status + tile), "l"(kIncl | (excl + tot))
                             : "memory");
        }
        if (lane == 0) *smem1 = excl;
    }
    __syncthreads();
    return *smem1;
}

// Exclusive u32 -> u64 scan, one 4096-element tile per block with decoupled
// look-back.  Inputs are read warp-striped (coalesced 128-byte rows) and transposed
// through shared memory so each thread scans 16 consecutive items; the u64 results
// go back through shared memory and leave warp-striped as well.
__global__ void __launch_bounds__(kThreads)
k_scan_u32(const std::uint32_t* __restrict__ in, std::uint64_t n, std::uint64_t* __restrict__ out,
           unsigned long long* status, std::uint32_t* ticket, std::uint64_t* total) {
    __shared__ std::uint64_t sm[40];
    __shared__ std::uint32_t s_tile;
    // shared staging with one pad word per 32 (conflict-free blocked and striped access)
    constexpr int kPad = kTile + kTile / 32;
    __shared__ std::uint64_t s_buf[kPad];  // u32 inputs (first half), then u64 outputs
    auto* s_in = reinterpret_cast<std::uint32_t*>(s_buf);
    auto pad = [](int i) { return i + (i >> 5); };
    if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
    __syncthreads();
    const std::uint32_t tile = s_tile;
    const std::uint64_t base = static_cast<std::uint64_t>(tile) * kTile;
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
        const std::uint64_t i = base + static_cast<std::uint64_t>(k) * kThreads + threadIdx.x;
        s_in[pad(k * kThreads + threadIdx.x)] = i < n ? in[i] : 0u;
    }
    __syncthreads();
    std::uint32_t v[kItems];
    std::uint64_t sum = 0;
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
        v[k] = s_in[pad(threadIdx.x * kItems + k)];
        sum += v[k];
    }
    std::uint64_t block_total;
    const std::uint64_t excl = block_excl_scan(sum, &block_total, sm);  // (ends with a barrier)
    const std::uint64_t prefix = tile_lookback1(status, tile, block_total, sm + 34);
    std::uint64_t at = prefix + excl;
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
        s_buf[pad(threadIdx.x * kItems + k)] = at;
        at += v[k];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
        const std::uint64_t i = base + static_cast<std::uint64_t>(k) * kThreads + threadIdx.x;
        if (i < n) out[i] = s_buf[pad(k * kThreads + threadIdx.x)];
    }
    const std::uint64_t ntiles = (n + kTile - 1) / kTile;
    if (tile == ntiles - 1 && threadIdx.x == 0 && total) *total = prefix + block_total;
}

__global__ void k_finite_f32(const float* v, std::uint64_t n, unsigned long long* bad) {
    for (std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<std::uint64_t>(gridDim.x) * blockDim.x)
        if (!isfinite(v[i])) atomicMin(bad, static_cast<unsigned long long>(i));
}
__global__ void k_finite_f64(const double* v, std::uint64_t n, unsigned long long* bad) {
    for (std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<std::uint64_t>(gridDim.x) * blockDim.x)
        if (!isfinite(v[i])) atomicMin(bad, static_cast<unsigned long long>(i));
}

__global__ void k_small_copy(const std::uint64_t* __restrict__ src, volatile std::uint64_t* dst, int n) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
}

}  // namespace

int launch_check_finite(const void* values, int value_type, std::uint64_t n, unsigned long long* first_bad,
                        cudaStream_t s, int num_sms) {
    if (n == 0) return MSC3D_OK;
    const unsigned grid = static_cast<unsigned>(std::min<std::uint64_t>((n + 255) / 256, 16ull * num_sms));
    if (value_type == MSC3D_VALUE_F64) k_finite_f64<<<grid, 256, 0, s>>>(static_cast<const double*>(values), n, first_bad);
    else k_finite_f32<<<grid, 256, 0, s>>>(static_cast<const float*>(values), n, first_bad);
    count_launch();
    MSC3D_CUDA_TRY(cudaGetLastError());
    return MSC3D_OK;
}

int launch_small_copy(const std::uint64_t* src, std::uint64_t* dst_mapped, int n, cudaStream_t s) {
    if (n <= 0) return MSC3D_OK;
    k_small_copy<<<1, 128, 0, s>>>(src, dst_mapped, n);
    count_launch();
    MSC3D_CUDA_TRY(cudaGetLastError());
    return MSC3D_OK;
}

int scan_u32(const std::uint32_t* in, std::uint64_t n, std::uint64_t* out, std::uint64_t* d_total,
             Workspace& ws, cudaStream_t s) {
    if (n == 0) {
        MSC3D_CUDA_TRY(cudaMemsetAsync(d_total, 0, 8, s));
        return MSC3D_OK;
    }
    const std::uint64_t ntiles = (n + kTile - 1) / kTile;
    char* buf = static_cast<char*>(ws.get(ntiles * 8 + 16));
    if (!buf) return MSC3D_ERR_NOMEM;
    auto* status = reinterpret_cast<unsigned long long*>(buf);
    auto* ticket = reinterpret_cast<std::uint32_t*>(status + ntiles);
    MSC3D_CUDA_TRY(cudaMemsetAsync(buf, 0, ntiles * 8 + 4, s));
    k_scan_u32<<<static_cast<unsigned>(ntiles), kThreads, 0, s>>>(in, n, out, status, ticket, d_total);
    count_launch();
    MSC3D_CUDA_TRY(cudaGetLastError());
    return MSC3D_OK;
}

}  // namespace msc3d_dev

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
constexpr int kItems = 8;
constexpr int kTile = kThreads * kItems;

__global__ void __launch_bounds__(kThreads)
k_scan_u32(const std::uint32_t* __restrict__ in, std::uint64_t n, std::uint64_t* __restrict__ out,
           TileStatus st, std::uint64_t* total) {
    __shared__ std::uint64_t sm[40];
    __shared__ std::uint32_t s_tile;
    if (threadIdx.x == 0) s_tile = atomicAdd(st.ticket, 1u);
    __syncthreads();
    const std::uint32_t tile = s_tile;
    const std::uint64_t first = static_cast<std::uint64_t>(tile) * kTile +
                                static_cast<std::uint64_t>(threadIdx.x) * kItems;
    std::uint32_t v[kItems];
    std::uint64_t sum = 0;
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
        v[k] = first + k < n ? in[first + k] : 0u;
        sum += v[k];
    }
    std::uint64_t block_total;
    const std::uint64_t excl = block_excl_scan(sum, &block_total, sm);
    const std::uint64_t tot[4] = {block_total, 0, 0, 0};
    tile_lookback4(st, tile, tot, sm + 34);
    std::uint64_t at = sm[34] + excl;
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
        if (first + k < n) out[first + k] = at;
        at += v[k];
    }
    const std::uint64_t ntiles = (n + kTile - 1) / kTile;
    if (tile == ntiles - 1 && threadIdx.x == 0 && total) *total = sm[34] + block_total;
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
    char* buf = static_cast<char*>(ws.get(ntiles * 68 + 16));
    if (!buf) return MSC3D_ERR_NOMEM;
    TileStatus st;
    st.agg = reinterpret_cast<std::uint64_t*>(buf);
    st.incl = st.agg + 4 * ntiles;
    st.flag = reinterpret_cast<std::uint32_t*>(st.incl + 4 * ntiles);
    st.ticket = st.flag + ntiles;
    MSC3D_CUDA_TRY(cudaMemsetAsync(st.flag, 0, (ntiles + 1) * 4, s));
    k_scan_u32<<<static_cast<unsigned>(ntiles), kThreads, 0, s>>>(in, n, out, st, d_total);
    count_launch();
    MSC3D_CUDA_TRY(cudaGetLastError());
    return MSC3D_OK;
}

}  // namespace msc3d_dev

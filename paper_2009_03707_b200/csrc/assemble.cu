// Device-side assembly of the MSComplex (proj/src/msc.cpp:89-145):
//   * critical points = concatenation of the four ascending lists (id = position);
//   * arcs min->1s, 1s->2s, 2s->max in critical-point ids, globally sorted by
//     (src, dst).  The 1s->2s block comes out of counting already sorted; the
//     2s->max block is generated per 2-saddle in order; only the min->1s block must
//     be transposed (grouped by minimum): counting scatter by minimum, then a
//     per-minimum sort of the (small) buckets.
//   * id translation helpers (rank -> cell, rank -> cp id).
#include "common.cuh"
#include "kernels.cuh"

namespace msc3d_dev {

namespace {

constexpr int kThreads = 256;

// One item per thread (the grid-stride loops below then run once): blocks are
// scheduled in id order, so the resident ones sweep the id space as a compact
// wavefront and spatially neighbouring items share the L2.
inline unsigned grid_for(std::uint64_t n, int /*num_sms*/, int /*per_sm*/ = 16) {
    return static_cast<unsigned>(std::max<std::uint64_t>(1, (n + kThreads - 1) / kThreads));
}

#define GRID_STRIDE(i, n)                                                                       \
    for (std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x; \
         i < (n); i += static_cast<std::uint64_t>(gridDim.x) * blockDim.x)

template <typename IdT>
__global__ void k_gather_ids(const IdT* __restrict__ list, const std::uint32_t* __restrict__ idx,
                             std::uint64_t n, IdT* __restrict__ out) {
    GRID_STRIDE(i, n) out[i] = list[idx[i]];
}

template <typename IdT>
__global__ void k_cp_concat(const IdT* __restrict__ src, std::uint64_t n, std::uint64_t at,
                            std::uint8_t index, IdT* __restrict__ cp_cell,
                            std::uint8_t* __restrict__ cp_index) {
    GRID_STRIDE(i, n) {
        cp_cell[at + i] = src[i];
        cp_index[at + i] = index;
    }
}

// Per 1-saddle k (cp id base1 + k): its minima via the vertex labels.
// Emits (min id, saddle id, mult) into two slots; counts per minimum.
template <typename IdT>
__global__ void k_arcs_min(const IdT* __restrict__ crit1, std::uint64_t n1, Dims d,
                           const std::uint32_t* __restrict__ label0, RankRemap remap0,
                           std::uint32_t base1, std::uint32_t* __restrict__ slot_min,
                           std::uint32_t* __restrict__ per_min) {
    GRID_STRIDE(k, n1) {
        const Coord c = unpack(d, crit1[k]);
        const int axis = (c.x & 1) ? 0 : ((c.y & 1) ? 1 : 2);
        Coord lo = c, hi = c;
        if (axis == 0) { lo.x -= 1; hi.x += 1; }
        else if (axis == 1) { lo.y -= 1; hi.y += 1; }
        else { lo.z -= 1; hi.z += 1; }
        const std::uint32_t a = remap0(label0[vertex_dense(d, lo)]);
        const std::uint32_t b = remap0(label0[vertex_dense(d, hi)]);
        if (a == b) {
            slot_min[2 * k] = a;
            slot_min[2 * k + 1] = kNoLabel;
            atomicAdd(&per_min[a], 1u);
        } else {
            slot_min[2 * k] = a < b ? a : b;
            slot_min[2 * k + 1] = a < b ? b : a;
            atomicAdd(&per_min[a], 1u);
            atomicAdd(&per_min[b], 1u);
        }
        (void)base1;
    }
}

// Scatter into minimum buckets: key = saddle id << 1 | (mult == 2).
// (The arc's source is its bucket's minimum whatever its place in the bucket, so it
// is written here; the sorted keys then give destinations and multiplicities.)
__global__ void k_arcs_min_scatter(const std::uint32_t* __restrict__ slot_min, std::uint64_t n1,
                                   std::uint32_t base1, const std::uint64_t* __restrict__ off,
                                   std::uint32_t* __restrict__ cursor, std::uint64_t* __restrict__ key,
                                   std::uint32_t* __restrict__ asrc) {
    GRID_STRIDE(k, n1) {
        const std::uint32_t a = slot_min[2 * k], b = slot_min[2 * k + 1];
        const std::uint64_t sid = base1 + k;
        if (b == kNoLabel) {
            const std::uint64_t at = off[a] + atomicAdd(&cursor[a], 1u);
            key[at] = (sid << 1) | 1ull;
            asrc[at] = a;
        } else {
            std::uint64_t at = off[a] + atomicAdd(&cursor[a], 1u);
            key[at] = sid << 1;
            asrc[at] = a;
            at = off[b] + atomicAdd(&cursor[b], 1u);
            key[at] = sid << 1;
            asrc[at] = b;
        }
    }
}

// Sort every bucket [off[m], off[m+1]) ascending.  Thread per bucket (insertion
// sort) for small buckets; large buckets are left for k_sort_large_buckets.
__global__ void k_sort_small_buckets(const std::uint64_t* __restrict__ off, std::uint64_t nb,
                                     std::uint64_t total, std::uint64_t* __restrict__ key,
                                     std::uint32_t* __restrict__ large, unsigned long long* n_large) {
    GRID_STRIDE(m, nb) {
        const std::uint64_t b = off[m], e = m + 1 < nb ? off[m + 1] : total;
        const std::uint64_t n = e - b;
        if (n <= 1) continue;
        if (n > 64) {
            large[atomicAdd(n_large, 1ull)] = static_cast<std::uint32_t>(m);
            continue;
        }
        if (n <= 8) {  // (most buckets) in registers: all loads first, an 8-input network
            std::uint64_t v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] = static_cast<std::uint64_t>(q) < n ? key[b + q] : ~0ull;
            auto ce = [](std::uint64_t& x, std::uint64_t& y) {
                const std::uint64_t lo = x < y ? x : y, hi = x < y ? y : x;
                x = lo;
                y = hi;
            };
            // Batcher odd-even merge sort, 19 comparators
            ce(v[0], v[1]); ce(v[2], v[3]); ce(v[4], v[5]); ce(v[6], v[7]);
            ce(v[0], v[2]); ce(v[1], v[3]); ce(v[4], v[6]); ce(v[5], v[7]);
            ce(v[1], v[2]); ce(v[5], v[6]);
            ce(v[0], v[4]); ce(v[1], v[5]); ce(v[2], v[6]); ce(v[3], v[7]);
            ce(v[2], v[4]); ce(v[3], v[5]);
            ce(v[1], v[2]); ce(v[3], v[4]); ce(v[5], v[6]);
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (static_cast<std::uint64_t>(q) < n) key[b + q] = v[q];
            continue;
        }
        for (std::uint64_t i = b + 1; i < e; ++i) {
            const std::uint64_t v = key[i];
            std::uint64_t j = i;
            while (j > b && key[j - 1] > v) {
                key[j] = key[j - 1];
                --j;
            }
            key[j] = v;
        }
    }
}

// One block per large bucket: bitonic sort in shared memory in chunks of 4096,
// then (if the bucket is larger) repeated block-level merges through global
// memory scratch.
constexpr int kChunk = 4096;

__device__ void block_bitonic(std::uint64_t* s, int n_pow2) {
    for (int k = 2; k <= n_pow2; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < n_pow2; i += blockDim.x) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const bool up = (i & k) == 0;
                    const std::uint64_t a = s[i], b = s[ixj];
                    if ((a > b) == up) {
                        s[i] = b;
                        s[ixj] = a;
                    }
                }
            }
            __syncthreads();
        }
    }
}

// One large bucket m, by the whole block (s: kChunk shared words).
__device__ __forceinline__ void sort_large_one(const std::uint64_t* __restrict__ off, std::uint64_t nb,
                                               std::uint64_t total, std::uint32_t m, std::uint64_t* __restrict__ key,
                                               std::uint64_t* __restrict__ scratch, std::uint64_t* s) {
    const std::uint64_t b = off[m], e = m + 1 < nb ? off[m + 1] : total;
    const std::uint64_t n = e - b;
    // 1) sort chunks
    for (std::uint64_t c0 = 0; c0 < n; c0 += kChunk) {
        const int cn = static_cast<int>(n - c0 < static_cast<std::uint64_t>(kChunk) ? n - c0 : static_cast<std::uint64_t>(kChunk));
        int p2 = 1;
        while (p2 < cn) p2 <<= 1;
        for (int i = threadIdx.x; i < p2; i += blockDim.x) s[i] = i < cn ? key[b + c0 + i] : ~0ull;
        __syncthreads();
        block_bitonic(s, p2);
        for (int i = threadIdx.x; i < cn; i += blockDim.x) key[b + c0 + i] = s[i];
        __syncthreads();
    }
    // 2) merge runs pairwise (runs of width w), ping-pong through scratch[b..e)
    std::uint64_t* src = key + b;
    std::uint64_t* dst = scratch + b;
    for (std::uint64_t w = kChunk; w < n; w <<= 1) {
        for (std::uint64_t r = 0; r < n; r += 2 * w) {
            const std::uint64_t lo = r, mid = min(r + w, n), hi = min(r + 2 * w, n);
            // each thread computes output positions of a subset of elements by
            // binary search in the other run (merge by rank; keys are unique)
            for (std::uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
                const std::uint64_t v = src[i];
                std::uint64_t rank;
                if (i < mid) {
                    std::uint64_t a = mid, z = hi;  // count of elements in right run < v
                    while (a < z) {
                        const std::uint64_t h = (a + z) >> 1;
                        if (src[h] < v) a = h + 1;
                        else z = h;
                    }
                    rank = (i - lo) + (a - mid);
                } else {
                    std::uint64_t a = lo, z = mid;  // elements in left run <= v
                    while (a < z) {
                        const std::uint64_t h = (a + z) >> 1;
                        if (src[h] <= v) a = h + 1;
                        else z = h;
                    }
                    rank = (i - mid) + (a - lo);
                }
                dst[lo + rank] = v;
            }
        }
        __syncthreads();
        std::uint64_t* t = src;
        src = dst;
        dst = t;
    }
    if (src != key + b)
        for (std::uint64_t i = threadIdx.x; i < n; i += blockDim.x) key[b + i] = src[i];
    __syncthreads();
}

__global__ void k_sort_large_buckets(const std::uint64_t* __restrict__ off, std::uint64_t nb,
                                     std::uint64_t total, const std::uint32_t* __restrict__ large,
                                     std::uint64_t* __restrict__ key, std::uint64_t* __restrict__ scratch) {
    __shared__ std::uint64_t s[kChunk];
    sort_large_one(off, nb, total, large[blockIdx.x], key, scratch, s);
}

// The same with the number of large buckets read on the device (no host round trip):
// blocks take buckets large[blockIdx.x + k * gridDim.x].
__global__ void k_sort_large_loop(const std::uint64_t* __restrict__ off, std::uint64_t nb, std::uint64_t total,
                                  const std::uint32_t* __restrict__ large, const unsigned long long* __restrict__ n_large,
                                  std::uint64_t* __restrict__ key, std::uint64_t* __restrict__ scratch) {
    __shared__ std::uint64_t s[kChunk];
    const unsigned long long nl = *n_large;
    for (unsigned long long k = blockIdx.x; k < nl; k += gridDim.x) sort_large_one(off, nb, total, large[k], key, scratch, s);
}

// Block A arcs out of the sorted buckets, one arc per thread: dst = saddle id, mult.
__global__ void k_arcs_min_emit(std::uint64_t total, const std::uint64_t* __restrict__ key,
                                std::uint32_t* __restrict__ adst, std::uint64_t* __restrict__ amult) {
    GRID_STRIDE(i, total) {
        const std::uint64_t k = key[i];
        adst[i] = static_cast<std::uint32_t>(k >> 1);
        amult[i] = (k & 1) ? 2ull : 1ull;
    }
}

// Block C: per 2-saddle k (cp id base2 + k), its maxima via the cube labels.
template <typename IdT>
__global__ void k_arcs_max(const IdT* __restrict__ crit2, std::uint64_t n2, Dims d,
                           const std::uint32_t* __restrict__ label3, RankRemap remap3,
                           std::uint32_t* __restrict__ slot, std::uint32_t* __restrict__ cnt) {
    GRID_STRIDE(k, n2) {
        const Coord c = unpack(d, crit2[k]);
        const int axis = !(c.x & 1) ? 0 : (!(c.y & 1) ? 1 : 2);
        const std::int64_t coord = axis == 0 ? c.x : (axis == 1 ? c.y : c.z);
        const std::int64_t ext = axis == 0 ? d.ex : (axis == 1 ? d.ey : d.ez);
        std::uint32_t got[2] = {kNoLabel, kNoLabel};
        int ng = 0;
        for (int sgn = -1; sgn <= 1; sgn += 2) {
            const std::int64_t nc = coord + sgn;
            if (nc < 0 || nc >= ext) continue;
            Coord o = c;
            if (axis == 0) o.x = nc;
            else if (axis == 1) o.y = nc;
            else o.z = nc;
            got[ng++] = remap3(label3[cube_dense(d, o)]);
        }
        const std::uint32_t a = got[0], b = got[1];
        std::uint32_t n = 0;
        if (a != kNoLabel && a == b) {
            slot[2 * k] = a | 0x80000000u;
            slot[2 * k + 1] = kNoLabel;
            n = 1;
        } else {
            const std::uint32_t x = a < b ? a : b, y = a < b ? b : a;
            slot[2 * k] = x;
            slot[2 * k + 1] = y;
            n = (x != kNoLabel) + (y != kNoLabel);
        }
        cnt[k] = n;
    }
}

__global__ void k_arcs_max_emit(const std::uint32_t* __restrict__ slot, std::uint64_t n2,
                                std::uint32_t base2, const std::uint64_t* __restrict__ off,
                                std::uint32_t* __restrict__ asrc, std::uint32_t* __restrict__ adst,
                                std::uint64_t* __restrict__ amult) {
    GRID_STRIDE(k, n2) {
        std::uint64_t at = off[k];
        for (int s = 0; s < 2; ++s) {
            const std::uint32_t v = slot[2 * k + s];
            if (v == kNoLabel) continue;
            asrc[at] = base2 + static_cast<std::uint32_t>(k);
            adst[at] = v & 0x7fffffffu;
            amult[at] = (v & 0x80000000u) ? 2ull : 1ull;
            ++at;
        }
    }
}

// Host delivery of multiplicities: one byte per arc (values <= vmax (254) as they are,
// 255 = "see the escape list"), the rest as (index, value) pairs appended in any order
// (warp-aggregated; ~1% of the 1s->2s arcs of a noisy field).  Appends past `cap` are
// counted but dropped: the host then copies the u64 array instead.
__global__ void k_pack_mult(const std::uint64_t* __restrict__ mult, std::uint64_t n, std::uint64_t vmax,
                            std::uint8_t* __restrict__ out8, ulonglong2* __restrict__ esc, std::uint64_t cap,
                            unsigned long long* __restrict__ n_esc) {
    const std::uint64_t stride = static_cast<std::uint64_t>(gridDim.x) * blockDim.x;
    for (std::uint64_t base = (blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x) & ~31ull; base < n;
         base += stride) {
        const std::uint64_t i = base + (threadIdx.x & 31);
        const std::uint64_t m = i < n ? mult[i] : 0;
        const bool big = i < n && m > vmax;
        if (i < n) out8[i] = static_cast<std::uint8_t>(big ? 255u : m);
        const unsigned ball = __ballot_sync(0xffffffffu, big);
        if (ball) {
            const int lane = threadIdx.x & 31, leader = __ffs(ball) - 1;
            unsigned long long at = 0;
            if (lane == leader) at = atomicAdd(n_esc, static_cast<unsigned long long>(__popc(ball)));
            at = __shfl_sync(0xffffffffu, at, leader) + __popc(ball & ((1u << lane) - 1u));
            if (big && at < cap) esc[at] = make_ulonglong2(i, m);
        }
    }
}

// Host delivery of a sorted u32 array (the arc sources): one byte per entry = the
// difference to the previous entry (<= vmax = 254), 255 = "absolute value in the escape list"
// (also any decrease: unsorted input stays exact), and the first entry of every chunk
// of kSrcChunk as a u32 head, so the host decodes the chunks independently.
constexpr std::uint64_t kSrcChunk = 1ull << 16;
__global__ void k_pack_src(const std::uint32_t* __restrict__ src, std::uint64_t n, std::uint32_t vmax,
                           std::uint8_t* __restrict__ out8,
                           std::uint32_t* __restrict__ heads, ulonglong2* __restrict__ esc, std::uint64_t cap,
                           unsigned long long* __restrict__ n_esc) {
    const std::uint64_t stride = static_cast<std::uint64_t>(gridDim.x) * blockDim.x;
    for (std::uint64_t base = (blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x) & ~31ull; base < n;
         base += stride) {
        const std::uint64_t i = base + (threadIdx.x & 31);
        bool big = false;
        if (i < n) {
            const std::uint32_t v = src[i];
            const bool head = (i & (kSrcChunk - 1)) == 0;
            const std::uint32_t prev = head ? v : src[i - 1];
            big = !head && (v < prev || v - prev > vmax);
            out8[i] = static_cast<std::uint8_t>(head ? 0u : (big ? 255u : v - prev));
            if (head) heads[i / kSrcChunk] = v;
        }
        const unsigned ball = __ballot_sync(0xffffffffu, big);
        if (ball) {
            const int lane = threadIdx.x & 31, leader = __ffs(ball) - 1;
            unsigned long long at = 0;
            if (lane == leader) at = atomicAdd(n_esc, static_cast<unsigned long long>(__popc(ball)));
            at = __shfl_sync(0xffffffffu, at, leader) + __popc(ball & ((1u << lane) - 1u));
            if (big && at < cap) esc[at] = make_ulonglong2(i, src[i]);
        }
    }
}

}  // namespace

int launch_gather_ids(const void* list, const std::uint32_t* idx, std::uint64_t n, int id_width,
                      void* out, cudaStream_t s, int num_sms) {
    if (n == 0) return MSC3D_OK;
    if (id_width == 4)
        k_gather_ids<std::uint32_t><<<grid_for(n, num_sms), kThreads, 0, s>>>(
            static_cast<const std::uint32_t*>(list), idx, n, static_cast<std::uint32_t*>(out));
    else
        k_gather_ids<std::uint64_t><<<grid_for(n, num_sms), kThreads, 0, s>>>(
            static_cast<const std::uint64_t*>(list), idx, n, static_cast<std::uint64_t*>(out));
    count_launch();
    MSC3D_CUDA_TRY(cudaGetLastError());
    return MSC3D_OK;
}

// CriticalPoint::value (msc.cpp:106): the sample at the cell's maximum vertex, the
// larger value and, on equal values, the larger id (max_vertex_of, grid.cpp:129-137),
// widened to double exactly.
template <typename IdT, typename T>
__global__ void k_cp_values(const IdT* __restrict__ cells, std::uint64_t n, Dims d, const T* __restrict__ f,
                            double* __restrict__ out) {
    GRID_STRIDE(i, n) {
        const Coord c = unpack(d, cells[i]);
        const std::int64_t x0 = c.x >> 1, y0 = c.y >> 1, z0 = c.z >> 1;
        const int dx = static_cast<int>(c.x & 1), dy = static_cast<int>(c.y & 1), dz = static_cast<int>(c.z & 1);
        T bv = T(0);
        std::int64_t bid = -1;
        for (int oz = 0; oz <= dz; ++oz)
            for (int oy = 0; oy <= dy; ++oy)
                for (int ox = 0; ox <= dx; ++ox) {
                    const std::int64_t vid = (x0 + ox) + d.nx * ((y0 + oy) + d.ny * (z0 + oz));
                    const T v = f[vid];
                    if (bid < 0 || v > bv || (v == bv && vid > bid)) {
                        bv = v;
                        bid = vid;
                    }
                }
        out[i] = static_cast<double>(bv);
    }
}

int launch_cp_values(const void* cells, int id_width, std::uint64_t n, const Dims& d, const void* values,
                     int value_type, double* out, cudaStream_t s, int num_sms) {
    if (n == 0) return MSC3D_OK;
    const unsigned g = grid_for(n, num_sms);
    if (value_type == MSC3D_VALUE_F64) {
        if (id_width == 4)
            k_cp_values<<<g, kThreads, 0, s>>>(static_cast<const std::uint32_t*>(cells), n, d,
                                               static_cast<const double*>(values), out);
        else
            k_cp_values<<<g, kThreads, 0, s>>>(static_cast<const std::uint64_t*>(cells), n, d,
                                               static_cast<const double*>(values), out);
    } else {
        if (id_width == 4)
            k_cp_values<<<g, kThreads, 0, s>>>(static_cast<const std::uint32_t*>(cells), n, d,
                                               static_cast<const float*>(values), out);
        else
            k_cp_values<<<g, kThreads, 0, s>>>(static_cast<const std::uint64_t*>(cells), n, d,
                                               static_cast<const float*>(values), out);
    }
    count_launch();
    MSC3D_CUDA_TRY(cudaGetLastError());
    return MSC3D_OK;
}

int launch_cp_concat(const void* src, std::uint64_t n, std::uint64_t at, int index, int id_width,
                     void* cp_cell, std::uint8_t* cp_index, cudaStream_t s, int num_sms) {
    if (n == 0) return MSC3D_OK;
    if (id_width == 4)
        k_cp_concat<std::uint32_t><<<grid_for(n, num_sms), kThreads, 0, s>>>(
            static_cast<const std::uint32_t*>(src), n, at, static_cast<std::uint8_t>(index),
            static_cast<std::uint32_t*>(cp_cell), cp_index);
    else
        k_cp_concat<std::uint64_t><<<grid_for(n, num_sms), kThreads, 0, s>>>(
            static_cast<const std::uint64_t*>(src), n, at, static_cast<std::uint8_t>(index),
            static_cast<std::uint64_t*>(cp_cell), cp_index);
    count_launch();
    MSC3D_CUDA_TRY(cudaGetLastError());
    return MSC3D_OK;
}

int launch_arcs_min(const void* crit1, std::uint64_t n1, int id_width, const Dims& d,
                    const std::uint32_t* label0, RankRemap remap0, std::uint32_t base1,
                    std::uint32_t* slot_min, std::uint32_t* per_min, cudaStream_t s, int num_sms) {
    if (n1 == 0) return MSC3D_OK;
    if (id_width == 4)
        k_arcs_min<std::uint32_t><<<grid_for(n1, num_sms), kThreads, 0, s>>>(
            static_cast<const std::uint32_t*>(crit1), n1, d, label0, remap0, base1, slot_min, per_min);
    else
        k_arcs_min<std::uint64_t><<<grid_for(n1, num_sms), kThreads, 0, s>>>(
            static_cast<const std::uint64_t*>(crit1), n1, d, label0, remap0, base1, slot_min, per_min);
    count_launch();
    MSC3D_CUDA_TRY(cudaGetLastError());
    return MSC3D_OK;
}

int launch_arcs_min_sort(const std::uint32_t* slot_min, std::uint64_t n1, std::uint32_t base1,
                         const std::uint64_t* off, std::uint64_t n0, std::uint64_t total,
                         std::uint32_t* cursor, std::uint64_t* key, std::uint64_t* scratch,
                         std::uint32_t* large, unsigned long long* n_large,
                         std::uint64_t* h_small, std::uint32_t* asrc, std::uint32_t* adst,
                         std::uint64_t* amult, cudaStream_t s, int num_sms) {
    if (n1 == 0) return MSC3D_OK;
    MSC3D_CUDA_TRY(cudaMemsetAsync(cursor, 0, n0 * 4, s));
    MSC3D_CUDA_TRY(cudaMemsetAsync(n_large, 0, 8, s));
    k_arcs_min_scatter<<<grid_for(n1, num_sms), kThreads, 0, s>>>(slot_min, n1, base1, off, cursor, key, asrc);
    k_sort_small_buckets<<<grid_for(n0, num_sms), kThreads, 0, s>>>(off, n0, total, key, large, n_large);
    count_launch(2);
    MSC3D_CUDA_TRY(cudaGetLastError());
    // large buckets: their count stays on the device (no host round trip: this chain runs
    // on a side stream beside the saddle stages)
    (void)h_small;
    k_sort_large_loop<<<static_cast<unsigned>(2 * num_sms), 512, 0, s>>>(off, n0, total, large, n_large, key, scratch);
    count_launch();
    k_arcs_min_emit<<<grid_for(total, num_sms), kThreads, 0, s>>>(total, key, adst, amult);
    count_launch();
    MSC3D_CUDA_TRY(cudaGetLastError());
    return MSC3D_OK;
}

// Sort every bucket [off[m], off[m+1]) (last bucket ends at `total`) of u64 keys
// ascending: thread-per-bucket insertion sort, block bitonic/merge for large ones.
int launch_bucket_sort(const std::uint64_t* off, std::uint64_t nb, std::uint64_t total,
                       std::uint64_t* key, std::uint64_t* scratch, std::uint32_t* large,
                       unsigned long long* n_large, std::uint64_t* h_small, cudaStream_t s, int num_sms) {
    if (nb == 0 || total == 0) return MSC3D_OK;
    MSC3D_CUDA_TRY(cudaMemsetAsync(n_large, 0, 8, s));
    k_sort_small_buckets<<<grid_for(nb, num_sms), kThreads, 0, s>>>(off, nb, total, key, large, n_large);
    count_launch();
    MSC3D_CUDA_TRY(cudaGetLastError());
    {  // kernel copy into the mapped host mirror (a DMA would queue behind bulk copies)
        std::uint64_t* hd = nullptr;
        MSC3D_CUDA_TRY(cudaHostGetDevicePointer(reinterpret_cast<void**>(&hd), h_small, 0));
        const int rc = launch_small_copy(reinterpret_cast<const std::uint64_t*>(n_large), hd, 1, s);
        if (rc != MSC3D_OK) return rc;
    }
    MSC3D_CUDA_TRY(cudaStreamSynchronize(s));
    if (h_small[0]) {
        k_sort_large_buckets<<<static_cast<unsigned>(h_small[0]), 512, 0, s>>>(off, nb, total, large, key, scratch);
        count_launch();
        MSC3D_CUDA_TRY(cudaGetLastError());
    }
    return MSC3D_OK;
}

int launch_arcs_max(const void* crit2, std::uint64_t n2, int id_width, const Dims& d,
                    const std::uint32_t* label3, RankRemap remap3, std::uint32_t* slot,
                    std::uint32_t* cnt, cudaStream_t s, int num_sms) {
    if (n2 == 0) return MSC3D_OK;
    if (id_width == 4)
        k_arcs_max<std::uint32_t><<<grid_for(n2, num_sms), kThreads, 0, s>>>(
            static_cast<const std::uint32_t*>(crit2), n2, d, label3, remap3, slot, cnt);
    else
        k_arcs_max<std::uint64_t><<<grid_for(n2, num_sms), kThreads, 0, s>>>(
            static_cast<const std::uint64_t*>(crit2), n2, d, label3, remap3, slot, cnt);
    count_launch();
    MSC3D_CUDA_TRY(cudaGetLastError());
    return MSC3D_OK;
}

int launch_arcs_max_emit(const std::uint32_t* slot, std::uint64_t n2, std::uint32_t base2,
                         const std::uint64_t* off, std::uint32_t* asrc, std::uint32_t* adst,
                         std::uint64_t* amult, cudaStream_t s, int num_sms) {
    if (n2 == 0) return MSC3D_OK;
    k_arcs_max_emit<<<grid_for(n2, num_sms), kThreads, 0, s>>>(slot, n2, base2, off, asrc, adst, amult);
    count_launch();
    MSC3D_CUDA_TRY(cudaGetLastError());
    return MSC3D_OK;
}

int launch_pack_mult(const std::uint64_t* mult, std::uint64_t n, std::uint64_t vmax, std::uint8_t* out8, void* esc,
                     std::uint64_t cap, unsigned long long* n_esc, cudaStream_t s, int num_sms) {
    if (vmax > 254) return MSC3D_ERR_INVALID;
    MSC3D_CUDA_TRY(cudaMemsetAsync(n_esc, 0, 8, s));
    if (n == 0) return MSC3D_OK;
    const unsigned grid = static_cast<unsigned>(std::min<std::uint64_t>((n + 255) / 256, 16ull * num_sms));
    k_pack_mult<<<grid, 256, 0, s>>>(mult, n, vmax, out8, static_cast<ulonglong2*>(esc), cap, n_esc);
    count_launch();
    MSC3D_CUDA_TRY(cudaGetLastError());
    return MSC3D_OK;
}

int launch_pack_src(const std::uint32_t* src, std::uint64_t n, std::uint64_t vmax, std::uint8_t* out8,
                    std::uint32_t* heads, void* esc, std::uint64_t cap, unsigned long long* n_esc, cudaStream_t s,
                    int num_sms) {
    if (vmax > 254) return MSC3D_ERR_INVALID;
    MSC3D_CUDA_TRY(cudaMemsetAsync(n_esc, 0, 8, s));
    if (n == 0) return MSC3D_OK;
    const unsigned grid = static_cast<unsigned>(std::min<std::uint64_t>((n + 255) / 256, 16ull * num_sms));
    k_pack_src<<<grid, 256, 0, s>>>(src, n, static_cast<std::uint32_t>(vmax), out8, heads, static_cast<ulonglong2*>(esc), cap,
                                    n_esc);
    count_launch();
    MSC3D_CUDA_TRY(cudaGetLastError());
    return MSC3D_OK;
}

std::uint64_t src_chunk() { return kSrcChunk; }

}  // namespace msc3d_dev

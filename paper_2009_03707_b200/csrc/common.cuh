// Shared device-side vocabulary for the msc3d B200 pipeline.
//
// Lattice conventions follow proj/include/msc3d/grid.hpp:8-23 (doubled
// coordinates, x-fastest ids, dimension = number of odd coordinates) and the
// pair-code byte of proj/include/msc3d/gradient.hpp:29-41.  Cell ids are 64-bit
// on the device; list outputs use IdT = uint32_t when the lattice has < 2^32
// cells (the reference's CellIndex, grid.hpp:33) and uint64_t beyond that.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/msc3d_cuda.h"

namespace msc3d_dev {

constexpr std::uint8_t kUnset = 0;
constexpr std::uint8_t kCritical = 1;
constexpr std::uint8_t kFacetBase = 2;
constexpr std::uint8_t kCofacetBase = 8;
constexpr std::uint32_t kNoLabel = 0xffffffffu;

// Division by a grid-invariant divisor with one 64x64->128 high multiply:
// q = umulhi(n, ceil(2^64 / d)), exact whenever n * d < 2^64 (ids < 2^36, d < 2^26
// here).  Replaces the 64-bit integer divisions of every id <-> coordinate map.
struct FastDiv {
    std::uint64_t d = 1, m = 0;
    __host__ __device__ static FastDiv make(std::uint64_t dv) {
        FastDiv f;
        f.d = dv;
        f.m = dv <= 1 ? 0 : (~0ull) / dv + 1;
        return f;
    }
    __host__ __device__ __forceinline__ std::uint64_t div(std::uint64_t n) const {
        if (d == 1) return n;
#ifdef __CUDA_ARCH__
        return __umul64hi(n, m);
#else
        return static_cast<std::uint64_t>((static_cast<unsigned __int128>(n) * m) >> 64);
#endif
    }
};

struct Dims {
    std::int64_t nx, ny, nz;   // vertices
    std::int64_t ex, ey, ez;   // lattice extents 2n-1
    std::int64_t exy;          // ex*ey
    std::uint64_t n_cells, n_verts, n_cubes;
    FastDiv fex, fey, fnx, fny, fmx, fmy;  // by ex, ey, nx, ny, nx-1, ny-1

    __host__ __device__ static Dims make(std::int64_t x, std::int64_t y, std::int64_t z) {
        Dims d;
        d.nx = x; d.ny = y; d.nz = z;
        d.ex = 2 * x - 1; d.ey = 2 * y - 1; d.ez = 2 * z - 1;
        d.exy = d.ex * d.ey;
        d.n_cells = static_cast<std::uint64_t>(d.ex) * d.ey * d.ez;
        d.n_verts = static_cast<std::uint64_t>(x) * y * z;
        d.n_cubes = static_cast<std::uint64_t>(x - 1) * (y - 1) * (z - 1);
        d.fex = FastDiv::make(d.ex);
        d.fey = FastDiv::make(d.ey);
        d.fnx = FastDiv::make(x);
        d.fny = FastDiv::make(y);
        d.fmx = FastDiv::make(x - 1);
        d.fmy = FastDiv::make(y - 1);
        return d;
    }
};

// Partner of a paired cell: one stride step along the encoded axis
// (gradient.hpp:51-60).
__host__ __device__ inline std::int64_t partner_of(const Dims& d, std::int64_t c, std::uint8_t k) {
    const int dir = k - (k < kCofacetBase ? kFacetBase : kCofacetBase);
    const int axis = dir >> 1;
    const std::int64_t step = axis == 0 ? 1 : (axis == 1 ? d.ex : d.exy);
    return (dir & 1) ? c + step : c - step;
}

__host__ __device__ inline bool paired_with_facet(std::uint8_t k) {
    return k >= kFacetBase && k < kCofacetBase;
}
__host__ __device__ inline bool paired_with_cofacet(std::uint8_t k) { return k >= kCofacetBase; }

struct Coord {
    std::int64_t x, y, z;
};

__host__ __device__ inline Coord unpack(const Dims& d, std::uint64_t id) {
    Coord c;
    const std::uint64_t q = d.fex.div(id);
    c.x = static_cast<std::int64_t>(id - q * d.ex);
    c.z = static_cast<std::int64_t>(d.fey.div(q));
    c.y = static_cast<std::int64_t>(q - static_cast<std::uint64_t>(c.z) * d.ey);
    return c;
}

__host__ __device__ inline std::uint64_t pack(const Dims& d, std::int64_t x, std::int64_t y,
                                              std::int64_t z) {
    return static_cast<std::uint64_t>(x + d.ex * (y + d.ey * z));
}

__host__ __device__ inline int cell_dim(const Coord& c) {
    return static_cast<int>((c.x & 1) + (c.y & 1) + (c.z & 1));
}

// Dense vertex / cube indices (proj/src/extrema.cpp:11-35).
__host__ __device__ inline std::uint32_t vertex_dense(const Dims& d, const Coord& c) {
    return static_cast<std::uint32_t>(c.x / 2 + d.nx * (c.y / 2 + d.ny * (c.z / 2)));
}
__host__ __device__ inline std::uint32_t cube_dense(const Dims& d, const Coord& c) {
    return static_cast<std::uint32_t>(c.x / 2 + (d.nx - 1) * (c.y / 2 + (d.ny - 1) * (c.z / 2)));
}
__host__ __device__ inline std::uint64_t vertex_cell(const Dims& d, std::uint64_t i) {
    const std::uint64_t r = d.fnx.div(i), x = i - r * d.nx, z = d.fny.div(r), y = r - z * d.ny;
    return pack(d, 2 * x, 2 * y, 2 * z);
}
__host__ __device__ inline std::uint64_t cube_cell(const Dims& d, std::uint64_t i) {
    const std::uint64_t mx = d.nx - 1, my = d.ny - 1;
    const std::uint64_t r = d.fmx.div(i), x = i - r * mx, z = d.fmy.div(r), y = r - z * my;
    return pack(d, 2 * x + 1, 2 * y + 1, 2 * z + 1);
}

}  // namespace msc3d_dev

namespace msc3d_dev {
// Kernel launches issued by this library (process-wide); bench.py reports it.
std::uint64_t& launch_counter();
inline void count_launch(std::uint64_t n = 1) { launch_counter() += n; }
}  // namespace msc3d_dev

#define MSC3D_CUDA_TRY(expr)                                              \
    do {                                                                  \
        cudaError_t _e = (expr);                                          \
        if (_e != cudaSuccess) return MSC3D_ERR_CUDA;                     \
    } while (0)

namespace msc3d_dev {
// Number of DAG successors of the edge at lattice coords (x, y, z)
// (saddle_graph.cpp:10-24): cofacet quads that are critical, or paired with a
// facet edge other than this one.
__device__ __forceinline__ int edge_successor_count(const std::uint8_t* __restrict__ codes, const Dims& d,
                                                    std::int64_t x, std::int64_t y, std::int64_t z) {
    const std::int64_t co[3] = {x, y, z};
    const std::int64_t ext[3] = {d.ex, d.ey, d.ez};
    const std::int64_t step[3] = {1, d.ex, d.exy};
    const std::int64_t e = x + d.ex * (y + d.ey * z);
    int n = 0;
#pragma unroll
    for (int b = 0; b < 3; ++b) {
        if (co[b] & 1) continue;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            if (h == 0 ? co[b] == 0 : co[b] == ext[b] - 1) continue;
            const std::int64_t q = e + (h ? step[b] : -step[b]);
            const std::uint8_t k = codes[q];
            if (k == kCritical) ++n;
            else if (paired_with_facet(k) && partner_of(d, q, k) != e) ++n;
        }
    }
    return n;
}
// Dense vertex/cube index -> critical point id through a bitmap of the critical
// extrema with one rank word per 32 entries (uint2 {rank of the word's first entry,
// bits}: 8 bytes per 32 vertices, L2-resident) instead of a 4-byte-per-entry id map
// gathered at random.  kNoLabel for entries whose bit is clear (non-critical roots).
struct RankRemap {
    const uint2* r;
    std::uint32_t base;
    __device__ __forceinline__ std::uint32_t operator()(std::uint32_t x) const {
        const uint2 w = r[x >> 5];
        const std::uint32_t b = 1u << (x & 31);
        return (w.y & b) ? base + w.x + static_cast<std::uint32_t>(__popc(w.y & (b - 1u))) : kNoLabel;
    }
};

}  // namespace msc3d_dev

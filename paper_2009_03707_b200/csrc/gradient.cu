// Lower-star discrete gradient on the B200 (assign_gradient, proj/src/gradient.cpp:79-283).
//
// One thread per vertex; the 3x3x3 vertex block around it is staged in shared
// memory once per CTA tile.  The reference's per-star work (27-slot arrays,
// per-cell sorted keys, two lazily-pruned queues) is restated as 27-bit slot
// masks:
//   * lower-star membership: the subset rule (gradient.cpp:104-120) evaluated as
//     two rounds of shifted mask ANDs;
//   * cell order key: the reference compares cells by their vertex values sorted
//     descending, then by vertex ids sorted descending, *independently*
//     (grid.cpp:91-122, gradient.cpp:53-63).  Inside one star this equals an
//     unsigned compare of ((value-thermometer mask) << 27 | vertex-slot mask):
//     the value part sets, for each vertex, the highest free bit at or below the
//     top rank of its equal-value group (so equal values compare as multisets),
//     the id part uses that ids of in-range neighbours increase with slot index;
//   * queues q0/q1 as masks; pop_min = argmin of the key over the mask; "number
//     of unassigned facets" = popcount(facet mask & ~assigned).
// Every cell is written exactly once, by the owner of its maximal vertex, so the
// scattered byte stores need no synchronisation.  Optionally the same kernel emits
// the two extremum forests (build_forest, extrema.cpp:43-77): a vertex's parent is
// the far end of the edge it pairs with, a cube's parent the cube across the quad
// it pairs with (itself at the boundary or when critical).
#include "common.cuh"
#include "kernels.cuh"

namespace msc3d_dev {

namespace {

struct SlotTables {
    std::int8_t off[27][3];
    std::uint8_t dim[27];
    std::uint32_t sub[27];      // vertex slots of the cell at slot t (incl. centre)
    std::uint32_t facet[27];    // facets of t that contain the centre vertex
    std::uint32_t cofacet[27];  // cofacets of t inside the 3x3x3 block
};

__constant__ SlotTables c_slot;

SlotTables host_tables() {
    SlotTables s{};
    for (int t = 0; t < 27; ++t) {
        const int o[3] = {t % 3 - 1, (t / 3) % 3 - 1, t / 9 - 1};
        for (int a = 0; a < 3; ++a) s.off[t][a] = static_cast<std::int8_t>(o[a]);
        s.dim[t] = static_cast<std::uint8_t>((o[0] != 0) + (o[1] != 0) + (o[2] != 0));
    }
    const int step[3] = {1, 3, 9};
    for (int t = 0; t < 27; ++t) {
        std::uint32_t sub = 0;
        for (int u = 0; u < 27; ++u) {
            bool ok = true;
            for (int a = 0; a < 3; ++a)
                ok = ok && (s.off[u][a] == 0 || s.off[u][a] == s.off[t][a]);
            if (ok) sub |= 1u << u;
        }
        s.sub[t] = sub;
        std::uint32_t fac = 0, cof = 0;
        for (int a = 0; a < 3; ++a) {
            if (s.off[t][a] != 0) fac |= 1u << (t - s.off[t][a] * step[a]);
            else {
                cof |= 1u << (t - step[a]);
                cof |= 1u << (t + step[a]);
            }
        }
        s.facet[t] = fac;
        s.cofacet[t] = cof;
    }
    return s;
}

constexpr int TX = 32, TY = 4, TZ = 2;
constexpr int SX = TX + 2, SY = TY + 2, SZ = TZ + 2;
constexpr std::uint32_t kCentre = 1u << 13;
constexpr std::uint32_t kAll = (1u << 27) - 1;

constexpr std::uint32_t axis_mask(int axis, int sign) {
    std::uint32_t m = 0;
    for (int t = 0; t < 27; ++t) {
        const int o = axis == 0 ? t % 3 - 1 : (axis == 1 ? (t / 3) % 3 - 1 : t / 9 - 1);
        if (o == sign) m |= 1u << t;
    }
    return m;
}
constexpr std::uint32_t kXP = axis_mask(0, 1), kXM = axis_mask(0, -1);
constexpr std::uint32_t kYP = axis_mask(1, 1), kYM = axis_mask(1, -1);
constexpr std::uint32_t kZP = axis_mask(2, 1), kZM = axis_mask(2, -1);
constexpr std::uint32_t kDim1 = (1u << 4) | (1u << 10) | (1u << 12) | (1u << 14) | (1u << 16) | (1u << 22);

__device__ __forceinline__ std::uint32_t facets_present(std::uint32_t s) {
    const std::uint32_t okx = (~(kXP | kXM) | ((s << 1) & kXP) | ((s >> 1) & kXM));
    const std::uint32_t oky = (~(kYP | kYM) | ((s << 3) & kYP) | ((s >> 3) & kYM));
    const std::uint32_t okz = (~(kZP | kZM) | ((s << 9) & kZP) | ((s >> 9) & kZM));
    return okx & oky & okz & kAll;
}

__device__ __forceinline__ int argmin_key(std::uint32_t m, const std::uint64_t* key) {
    int best = __ffs(m) - 1;
    std::uint64_t bk = key[best];
    m &= m - 1;
    while (m) {
        const int t = __ffs(m) - 1;
        m &= m - 1;
        if (key[t] < bk) {
            bk = key[t];
            best = t;
        }
    }
    return best;
}

template <typename T>
__global__ void __launch_bounds__(TX * TY * TZ)
k_gradient(const T* __restrict__ f, Dims d, std::uint8_t* __restrict__ codes,
           std::uint32_t* __restrict__ parent0, std::uint32_t* __restrict__ parent3) {
    __shared__ T tile[SZ][SY][SX];
    const std::int64_t x0 = static_cast<std::int64_t>(blockIdx.x) * TX - 1;
    const std::int64_t y0 = static_cast<std::int64_t>(blockIdx.y) * TY - 1;
    const std::int64_t z0 = static_cast<std::int64_t>(blockIdx.z) * TZ - 1;
    const int tid = threadIdx.x + TX * (threadIdx.y + TY * threadIdx.z);
    for (int i = tid; i < SX * SY * SZ; i += TX * TY * TZ) {
        const int lx = i % SX, ly = (i / SX) % SY, lz = i / (SX * SY);
        const std::int64_t gx = x0 + lx, gy = y0 + ly, gz = z0 + lz;
        T v = T(0);
        if (gx >= 0 && gx < d.nx && gy >= 0 && gy < d.ny && gz >= 0 && gz < d.nz)
            v = f[gx + d.nx * (gy + d.ny * gz)];
        tile[lz][ly][lx] = v;
    }
    __syncthreads();

    const std::int64_t vx = x0 + 1 + threadIdx.x, vy = y0 + 1 + threadIdx.y,
                       vz = z0 + 1 + threadIdx.z;
    if (vx >= d.nx || vy >= d.ny || vz >= d.nz) return;
    const T* base = &tile[threadIdx.z + 1][threadIdx.y + 1][threadIdx.x + 1];
    auto val = [&](int t) {
        return base[(t / 9 - 1) * (SX * SY) + ((t / 3) % 3 - 1) * SX + (t % 3 - 1)];
    };

    // In-range neighbours and "below the centre" in (value, id) order
    // (gradient.cpp:86-102); ids grow with slot index, so id < vi <=> slot < 13.
    std::uint32_t inr = kAll;
    if (vx == 0) inr &= ~kXM;
    if (vx == d.nx - 1) inr &= ~kXP;
    if (vy == 0) inr &= ~kYM;
    if (vy == d.ny - 1) inr &= ~kYP;
    if (vz == 0) inr &= ~kZM;
    if (vz == d.nz - 1) inr &= ~kZP;
    const T fv = val(13);
    std::uint32_t below = kCentre;
#pragma unroll
    for (int t = 0; t < 27; ++t) {
        if (t == 13) continue;
        const T u = val(t);
        if (u < fv || (u == fv && t < 13)) below |= 1u << t;
    }
    std::uint32_t S = below & inr;
    S &= facets_present(S);
    S &= facets_present(S);

    const std::int64_t vi = vx + d.nx * (vy + d.ny * vz);
    const std::int64_t vcell = 2 * vx + d.ex * (2 * vy + d.ey * 2 * vz);
    const std::int64_t sstep[3] = {1, d.ex, d.exy};
    auto cell_of = [&](int t) {
        return vcell + c_slot.off[t][0] + c_slot.off[t][1] * d.ex + c_slot.off[t][2] * d.exy;
    };

    if (S == kCentre) {  // |star| == 1: critical minimum (gradient.cpp:128-131)
        codes[vcell] = kCritical;
        if (parent0) parent0[vi] = static_cast<std::uint32_t>(vi);
        return;
    }

    // Top rank of each star vertex's equal-value group.
    std::uint8_t top[27];
    for (std::uint32_t m = S; m; m &= m - 1) {
        const int s = __ffs(m) - 1;
        const T vs = val(s);
        int c = -1;
        for (std::uint32_t n = S; n; n &= n - 1) c += val(__ffs(n) - 1) <= vs;
        top[s] = static_cast<std::uint8_t>(c);
    }
    std::uint64_t key[27];
    for (std::uint32_t m = S & ~kCentre; m; m &= m - 1) {
        const int t = __ffs(m) - 1;
        std::uint32_t vm = 0;
        for (std::uint32_t n = c_slot.sub[t]; n; n &= n - 1) {
            int b = top[__ffs(n) - 1];
            while ((vm >> b) & 1u) --b;
            vm |= 1u << b;
        }
        key[t] = (static_cast<std::uint64_t>(vm) << 27) | c_slot.sub[t];
    }

    auto write_pair = [&](int lo, int hi) {  // gradient.cpp:162-174
        int ax = 0;
        while (c_slot.off[lo][ax] == c_slot.off[hi][ax]) ++ax;
        const int sign = c_slot.off[hi][ax] - c_slot.off[lo][ax];
        codes[cell_of(lo)] = static_cast<std::uint8_t>(kCofacetBase + ax * 2 + (sign > 0));
        codes[cell_of(hi)] = static_cast<std::uint8_t>(kFacetBase + ax * 2 + (sign < 0));
        if (parent3 && c_slot.dim[hi] == 3) {
            // Cube hi pairs with quad lo; continue into the cube across lo
            // (extrema.cpp:63-75), or stop at a boundary quad.
            const int across = lo - (hi - lo);
            const std::int64_t cx = 2 * vx + c_slot.off[hi][0], cy = 2 * vy + c_slot.off[hi][1],
                               cz = 2 * vz + c_slot.off[hi][2];
            const std::uint32_t self =
                static_cast<std::uint32_t>(cx / 2 + (d.nx - 1) * (cy / 2 + (d.ny - 1) * (cz / 2)));
            std::uint32_t par = self;
            if ((inr >> across) & 1u) {
                const std::int64_t ax2 = 2 * vx + c_slot.off[across][0],
                                   ay2 = 2 * vy + c_slot.off[across][1],
                                   az2 = 2 * vz + c_slot.off[across][2];
                par = static_cast<std::uint32_t>(ax2 / 2 + (d.nx - 1) * (ay2 / 2 + (d.ny - 1) * (az2 / 2)));
            }
            parent3[self] = par;
        }
        (void)sstep;
    };

    std::uint32_t assigned = 0, q0 = 0, q1 = 0;
    auto settle = [&](int t) {  // gradient.cpp:178-193
        assigned |= 1u << t;
        for (std::uint32_t m = c_slot.cofacet[t] & S & ~assigned; m; m &= m - 1) {
            const int c = __ffs(m) - 1;
            if (__popc(c_slot.facet[c] & ~assigned) == 1) q1 |= 1u << c;
        }
    };

    // The vertex pairs with its lowest edge; other edges become candidates
    // (gradient.cpp:196-207).
    const std::uint32_t edges = S & kDim1;
    const int delta = argmin_key(edges, key);
    q0 = edges & ~(1u << delta);
    write_pair(13, delta);
    if (parent0) {
        parent0[vi] = static_cast<std::uint32_t>(vi + c_slot.off[delta][0] +
                                                 c_slot.off[delta][1] * d.nx +
                                                 c_slot.off[delta][2] * d.nx * d.ny);
    }
    settle(13);
    settle(delta);

    int remaining = __popc(S) - 2;
    while (remaining > 0) {  // gradient.cpp:226-264
        bool worked = false;
        for (;;) {
            const std::uint32_t cand = q1 & ~assigned;
            if (!cand) break;
            const int t = argmin_key(cand, key);
            q1 &= ~(1u << t);
            const std::uint32_t free_facets = c_slot.facet[t] & ~assigned;
            if (__popc(free_facets) != 1) {
                q0 |= 1u << t;
                continue;
            }
            const int fs = __ffs(free_facets) - 1;
            write_pair(fs, t);
            settle(fs);
            settle(t);
            remaining -= 2;
            worked = true;
        }
        if (remaining == 0) break;
        const std::uint32_t cand = q0 & ~assigned;
        if (cand) {
            const int t = argmin_key(cand, key);
            q0 &= ~(1u << t);
            codes[cell_of(t)] = kCritical;
            if (parent3 && c_slot.dim[t] == 3) {
                const std::int64_t cx = 2 * vx + c_slot.off[t][0], cy = 2 * vy + c_slot.off[t][1],
                                   cz = 2 * vz + c_slot.off[t][2];
                const std::uint32_t self = static_cast<std::uint32_t>(
                    cx / 2 + (d.nx - 1) * (cy / 2 + (d.ny - 1) * (cz / 2)));
                parent3[self] = self;
            }
            settle(t);
            --remaining;
            worked = true;
        }
        if (!worked) break;  // cannot happen on a valid star (gradient.cpp:259-262)
    }
}

bool g_tables_ready[64] = {false};

}  // namespace

int upload_gradient_tables(int device) {
    if (device >= 0 && device < 64 && g_tables_ready[device]) return MSC3D_OK;
    const SlotTables t = host_tables();
    MSC3D_CUDA_TRY(cudaMemcpyToSymbol(c_slot, &t, sizeof t));
    if (device >= 0 && device < 64) g_tables_ready[device] = true;
    return MSC3D_OK;
}

int launch_gradient(const void* values, int value_type, const Dims& d, std::uint8_t* codes,
                    std::uint32_t* parent0, std::uint32_t* parent3, cudaStream_t stream) {
    int dev = 0;
    MSC3D_CUDA_TRY(cudaGetDevice(&dev));
    const int rc = upload_gradient_tables(dev);
    if (rc != MSC3D_OK) return rc;
    const dim3 block(TX, TY, TZ);
    const dim3 grid(static_cast<unsigned>((d.nx + TX - 1) / TX),
                    static_cast<unsigned>((d.ny + TY - 1) / TY),
                    static_cast<unsigned>((d.nz + TZ - 1) / TZ));
    if (value_type == MSC3D_VALUE_F64)
        k_gradient<double><<<grid, block, 0, stream>>>(static_cast<const double*>(values), d,
                                                        codes, parent0, parent3);
    else
        k_gradient<float><<<grid, block, 0, stream>>>(static_cast<const float*>(values), d,
                                                      codes, parent0, parent3);
    count_launch();
    MSC3D_CUDA_TRY(cudaGetLastError());
    return MSC3D_OK;
}

}  // namespace msc3d_dev

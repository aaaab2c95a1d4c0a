// Lower-star discrete gradient on the B200 (assign_gradient, proj/src/gradient.cpp:79-283).
//
// One CTA stages a 32x4x2 vertex tile (+1 halo) in shared memory; each vertex's
// lower star is processed as 27-bit slot masks (slot t = (dx+1) + 3(dy+1) + 9(dz+1)):
//   * membership: the subset rule (gradient.cpp:104-120) as two rounds of shifted
//     mask ANDs;
//   * cell order (grid.cpp:91-122, gradient.cpp:53-63): cells are compared by their
//     vertex values sorted descending, then by vertex ids sorted descending,
//     *independently*.  With the star's vertices ranked by value (distinct values),
//     that is exactly an unsigned compare of the cells' rank bitmasks M(t)
//     (the larger maximum of the symmetric difference wins; a prefix loses);
//   * queues q0/q1 and "unassigned facets" as masks (popcount of facets & ~assigned),
//     pop_min = the cell of least rank mask.
//
// Fast path: the star's vertices are compacted into K registers, sorted by a
// bitonic network, ranked; every cell's rank mask is built from its facets' masks
// (unrolled over the 26 slots, constant indices) into a per-thread shared-memory
// column; the expansion pops the candidate of least mask (candidate sets are small).  The tile kernel
// runs stars of <= 8 cells (K = 8); larger stars are appended to two work lists
// processed by K = 16 / K = 32 kernels, whose register budgets do not cap the tile
// kernel's occupancy and whose warps are size-homogeneous.
//
// Stars containing two equal values go to the slow path (k_gradient_deferred),
// which keeps the reference's general multiset-then-ids key (value thermometer
// << 27 | vertex-slot mask): equal values compare as multisets, the id part uses
// that ids of in-range neighbours increase with slot index.
//
// Every cell is written exactly once, by the owner of its maximal vertex (plain
// byte stores).  The same kernel emits both extremum forests (build_forest,
// extrema.cpp:43-77) and the per-dimension critical counts.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"
#include "sortnet.cuh"

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

// Octant stars.  A lower star that is exactly one unit cube at the vertex (v, 3 edges,
// 3 quads, 1 cube -- 93% of the vertices of a smooth field) is paired by Robins'
// expansion according to the order of its 7 link vertices alone (distinct values;
// ties take the general path).  g_oct[Lehmer index of that order] holds the result
// for the canonical orientation (the cube at +x+y+z): for local cell m (bit a set =
// the cell spans axis a; 0 = v, 7 = the cube) two bits = partner axis + 1, 0 = critical.
// Reflections map the canonical result onto the other 7 orientations (with distinct
// values the expansion only compares cells, so it commutes with the reflection).
constexpr int kOctPerms = 5040;
__device__ std::uint16_t g_oct[kOctPerms];

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
            for (int a = 0; a < 3; ++a) ok = ok && (s.off[u][a] == 0 || s.off[u][a] == s.off[t][a]);
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

// Robins' expansion (gradient.cpp:196-264) on the canonical octant star for every
// order of its link vertices: cells compare by their rank masks.
std::vector<std::uint16_t> host_octant_table() {
    std::vector<std::uint16_t> table(kOctPerms);
    int perm[7] = {0, 1, 2, 3, 4, 5, 6};  // perm[i-1] = rank of link vertex i (local index 1..7)
    const int fact[7] = {720, 120, 24, 6, 2, 1, 1};
    do {
        int idx = 0;
        for (int i = 0; i < 7; ++i) {
            int c = 0;
            for (int j = i + 1; j < 7; ++j) c += perm[j] < perm[i];
            idx += c * fact[i];
        }
        std::uint32_t M[8];
        for (int m = 0; m < 8; ++m) {
            M[m] = 1u << 7;  // v: the largest
            for (int i = 1; i < 8; ++i)
                if ((i & m) == i) M[m] |= 1u << perm[i - 1];
        }
        auto facets = [](int m) {
            std::uint32_t f = 0;
            for (int a = 0; a < 3; ++a)
                if (m >> a & 1) f |= 1u << (m ^ (1 << a));
            return f;
        };
        auto cofacets = [](int m) {
            std::uint32_t f = 0;
            for (int a = 0; a < 3; ++a)
                if (!(m >> a & 1)) f |= 1u << (m | (1 << a));
            return f;
        };
        auto argmin = [&](std::uint32_t set) {
            int best = -1;
            for (int m = 0; m < 8; ++m)
                if ((set >> m & 1) && (best < 0 || M[m] < M[best])) best = m;
            return best;
        };
        std::uint32_t assigned = 0, q0 = 0, q1 = 0;
        int partner[8];
        for (int m = 0; m < 8; ++m) partner[m] = -2;
        auto settle = [&](int t) {
            assigned |= 1u << t;
            for (int c = 0; c < 8; ++c)
                if ((cofacets(t) >> c & 1) && !(assigned >> c & 1) &&
                    __builtin_popcount(facets(c) & ~assigned) == 1)
                    q1 |= 1u << c;
        };
        const int delta = argmin(0x16u);  // edges 1, 2, 4
        q0 = 0x16u & ~(1u << delta);
        partner[0] = delta;
        partner[delta] = 0;
        settle(0);
        settle(delta);
        int remaining = 6;
        while (remaining > 0) {
            for (;;) {
                const std::uint32_t cand = q1 & ~assigned;
                if (!cand) break;
                const int t = argmin(cand);
                q1 &= ~(1u << t);
                const std::uint32_t fr = facets(t) & ~assigned;
                if (__builtin_popcount(fr) != 1) {
                    q0 |= 1u << t;
                    continue;
                }
                const int f = __builtin_ctz(fr);
                partner[t] = f;
                partner[f] = t;
                settle(f);
                settle(t);
                remaining -= 2;
            }
            if (!remaining) break;
            const int t = argmin(q0 & ~assigned);
            q0 &= ~(1u << t);
            partner[t] = -1;
            settle(t);
            --remaining;
        }
        std::uint16_t e = 0;
        for (int m = 0; m < 8; ++m)
            if (partner[m] >= 0) e |= static_cast<std::uint16_t>((__builtin_ctz(m ^ partner[m]) + 1) << (2 * m));
        table[idx] = e;
    } while (std::next_permutation(perm, perm + 7));
    return table;
}

constexpr int TX = 32, TY = 4, TZ = 2;
constexpr int NT = TX * TY * TZ;
// A tile row in shared memory starts XO = 4 columns left of the tile's first vertex
// (the halo column is column 3) and is SX = 40 wide: the TMA box of the f32 tile loads
// (k_gradient<float, true>) must start at a 16-byte aligned x offset and span a multiple
// of 16 bytes.
constexpr int XO = 4;
constexpr int SX = TX + 2 * XO, SY = TY + 2, SZ = TZ + 2;
constexpr unsigned kTileBytesF32 = SX * SY * SZ * 4;  // 3840 = 30 x 128 (TMA destinations stay 128-B aligned)
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
constexpr std::uint32_t kDim3 = (1u << 0) | (1u << 2) | (1u << 6) | (1u << 8) | (1u << 18) | (1u << 20) |
                                (1u << 24) | (1u << 26);

constexpr int slot_off(int t, int a) { return a == 0 ? t % 3 - 1 : (a == 1 ? (t / 3) % 3 - 1 : t / 9 - 1); }
constexpr int slot_dim(int t) {
    return (slot_off(t, 0) != 0) + (slot_off(t, 1) != 0) + (slot_off(t, 2) != 0);
}
constexpr int slot_tile(int t) { return slot_off(t, 2) * (SX * SY) + slot_off(t, 1) * SX + slot_off(t, 0); }

__device__ __forceinline__ std::uint32_t facets_present(std::uint32_t s) {
    const std::uint32_t okx = (~(kXP | kXM) | ((s << 1) & kXP) | ((s >> 1) & kXM));
    const std::uint32_t oky = (~(kYP | kYM) | ((s << 3) & kYP) | ((s >> 3) & kYM));
    const std::uint32_t okz = (~(kZP | kZM) | ((s << 9) & kZP) | ((s >> 9) & kZM));
    return okx & oky & okz & kAll;
}

// slot -> offset in the shared tile (dynamic slot)
__device__ __forceinline__ int tile_off(int t) {
    const int z = (t * 57) >> 9;  // t / 9 for t < 27
    const int r = t - 9 * z;
    const int y = (r * 11) >> 5;  // r / 3 for r < 9
    const int x = r - 3 * y;
    return (z - 1) * (SX * SY) + (y - 1) * SX + (x - 1);
}

// Order-preserving unsigned key of a sample value (+0 and -0 compare equal).
__device__ __forceinline__ std::uint32_t ord_key(float v) {
    const std::uint32_t u = __float_as_uint(v + 0.0f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ std::uint64_t ord_key(double v) {
    const std::uint64_t u = static_cast<std::uint64_t>(__double_as_longlong(v + 0.0));
    return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}
template <typename T>
struct KeyOf;
template <>
struct KeyOf<float> {
    using type = std::uint32_t;
};
template <>
struct KeyOf<double> {
    using type = std::uint64_t;
};

constexpr std::uint32_t kX0 = kAll & ~(kXP | kXM), kY0 = kAll & ~(kYP | kYM), kZ0 = kAll & ~(kZP | kZM);

// 5-bit fields indexed by slot (0..26) in three 64-bit words.
struct Pack5 {
    std::uint64_t w[3] = {0, 0, 0};
    __device__ __forceinline__ void set(int slot, std::uint32_t v) {
        const int wi = slot >= 24 ? 2 : (slot >= 12 ? 1 : 0);
        const std::uint64_t x = static_cast<std::uint64_t>(v) << (5 * (slot - 12 * wi));
        if (wi == 0) w[0] |= x;
        else if (wi == 1) w[1] |= x;
        else w[2] |= x;
    }
    __device__ __forceinline__ std::uint32_t get(int slot) const {
        const int wi = slot >= 24 ? 2 : (slot >= 12 ? 1 : 0);
        const std::uint64_t ww = wi == 0 ? w[0] : (wi == 1 ? w[1] : w[2]);
        return static_cast<std::uint32_t>(ww >> (5 * (slot - 12 * wi))) & 31u;
    }
};

// Dense-id offset of the cube at slot t from the cube at slot 0 of a star.
__device__ __forceinline__ std::uint32_t cube_slot_offset(int t, const Dims& d) {
    const int z = t / 9, y = (t / 3) % 3, x = t % 3;
    return (x != 0 ? 1u : 0u) + (y != 0 ? static_cast<std::uint32_t>(d.nx - 1) : 0u) +
           (z != 0 ? static_cast<std::uint32_t>((d.nx - 1) * (d.ny - 1)) : 0u);
}

// Output side of one star: codes, forests, critical counts.
struct StarWriter {
    std::uint8_t* cbase;           // codes + vertex cell id
    const std::int32_t* cell_off;  // lattice offset per slot
    std::uint32_t* parent0;
    std::uint32_t* parent3;
    Dims d;
    std::int64_t vx, vy, vz;
    std::uint32_t inr;
    std::uint64_t ncrit;           // 16 bits per dimension

    std::uint32_t cube0, csy, csz;  // dense id of the cube at slot 0 (mod 2^32), cube strides

    __device__ __forceinline__ void init_cubes() {
        csy = static_cast<std::uint32_t>(d.nx - 1);
        csz = static_cast<std::uint32_t>((d.nx - 1) * (d.ny - 1));
        cube0 = static_cast<std::uint32_t>(vx - 1) + csy * static_cast<std::uint32_t>(vy - 1) +
                csz * static_cast<std::uint32_t>(vz - 1);
    }
    // dense id of the in-box cube at slot t (u32 wrap-around is exact: the result is)
    const std::uint32_t* cube_off;  // per slot: (x != 0) + (y != 0) * csy + (z != 0) * csz (block table)
    __device__ __forceinline__ std::uint32_t cube_dense_of(int t) const { return cube0 + cube_off[t]; }
    __device__ __forceinline__ void pair(int lo, int hi) {  // gradient.cpp:162-174
        const int diff = hi - lo;  // +-1, +-3 or +-9
        const int ad = diff < 0 ? -diff : diff;
        const int ax = ad == 1 ? 0 : (ad == 3 ? 1 : 2);
        const int pos = diff > 0;
        cbase[cell_off[lo]] = static_cast<std::uint8_t>(kCofacetBase + ax * 2 + pos);
        cbase[cell_off[hi]] = static_cast<std::uint8_t>(kFacetBase + ax * 2 + (1 - pos));
        if (lo == 13 && parent0) {
            const std::int64_t vi = vx + d.nx * (vy + d.ny * vz);
            const std::int64_t step = ax == 0 ? 1 : (ax == 1 ? d.nx : d.nx * d.ny);
            parent0[vi] = static_cast<std::uint32_t>(pos ? vi + step : vi - step);
        }
        if (parent3 && ((kDim3 >> hi) & 1u)) {
            // cube hi pairs with quad lo: continue into the cube across lo
            const int across = lo - diff;
            const std::uint32_t self = cube_dense_of(hi);
            parent3[self] = ((inr >> across) & 1u) ? cube_dense_of(across) : self;
        }
    }
    __device__ __forceinline__ void critical(int t, int dm) {
        cbase[cell_off[t]] = kCritical;
        ncrit += 1ull << (16 * dm);
        if (parent3 && dm == 3) {
            const std::uint32_t self = cube_dense_of(t);
            parent3[self] = self;
        }
    }
    __device__ __forceinline__ void minimum() {
        cbase[0] = kCritical;
        ncrit += 1ull;
        const std::int64_t vi = vx + d.nx * (vy + d.ny * vz);
        if (parent0) parent0[vi] = static_cast<std::uint32_t>(vi);
    }
};

// The lower-star expansion (gradient.cpp:196-264) over slot masks; `argmin`
// returns the least cell of a non-empty slot mask.
template <typename ArgMin>
__device__ __forceinline__ void robins(std::uint32_t S, const std::uint32_t* fac, const std::uint32_t* cof,
                                       ArgMin argmin, StarWriter& w) {
    std::uint32_t assigned = 0, q0 = 0, q1 = 0;
    // Bit-parallel unassigned-facet counts: a star cell's facets (those containing the
    // vertex) are its neighbours towards the centre along its non-centre coordinates,
    // so "facet along x unassigned" for all cells at once is a shift of the unassigned
    // mask by one slot (3 for y, 9 for z) under the masks of slots with x = 0 / x = 2.
    auto one_unassigned = [&](std::uint32_t U) {
        constexpr std::uint32_t X0 = 0x1249249u, X2 = X0 << 2;      // slots with x = 0 / 2
        constexpr std::uint32_t Y0 = 0x01c0e07u, Y2 = Y0 << 6;      // y = 0 / 2
        constexpr std::uint32_t Z0 = 0x00001ffu, Z2 = Z0 << 18;     // z = 0 / 2
        const std::uint32_t ux = ((U >> 1) & X0) | ((U << 1) & X2);
        const std::uint32_t uy = ((U >> 3) & Y0) | ((U << 3) & Y2);
        const std::uint32_t uz = ((U >> 9) & Z0) | ((U << 9) & Z2);
        return (ux ^ uy ^ uz) & ~(ux & uy & uz);  // exactly one unassigned facet
    };
    // (gradient.cpp:208-218: the in-star cofacets of t whose unassigned-facet count
    // drops to 1 join q1)
    auto settle = [&](int t) {
        assigned |= 1u << t;
        q1 |= cof[t] & S & ~assigned & one_unassigned(S & ~assigned);
    };
    const std::uint32_t edges = S & kDim1;
    const int delta = argmin(edges);
    q0 = edges & ~(1u << delta);
    w.pair(13, delta);
    settle(13);
    settle(delta);
    int remaining = __popc(S) - 2;
    while (remaining > 0) {
        bool worked = false;
        for (;;) {
            const std::uint32_t cand = q1 & ~assigned;
            if (!cand) break;
            const int t = argmin(cand);
            q1 &= ~(1u << t);
            const std::uint32_t free_f = fac[t] & ~assigned;
            if (__popc(free_f) != 1) {
                q0 |= 1u << t;
                continue;
            }
            const int fs = __ffs(free_f) - 1;
            w.pair(fs, t);
            settle(fs);
            settle(t);
            remaining -= 2;
            worked = true;
        }
        if (remaining == 0) break;
        const std::uint32_t cand = q0 & ~assigned;
        if (cand) {
            const int t = argmin(cand);
            q0 &= ~(1u << t);
            const int nf = __popc(fac[t]);  // dimension = number of v-containing facets
            w.critical(t, nf);
            settle(t);
            --remaining;
            worked = true;
        }
        if (!worked) break;  // cannot happen on a valid star (gradient.cpp:259-262)
    }
}

template <typename KT>
__device__ __forceinline__ void ce_pair(KT& ka, std::uint32_t& sa, KT& kb, std::uint32_t& sb, bool up) {
    const bool sw = up ? (kb < ka) : (ka < kb);
    const KT k0 = sw ? kb : ka, k1 = sw ? ka : kb;
    const std::uint32_t s0 = sw ? sb : sa, s1 = sw ? sa : sb;
    ka = k0;
    kb = k1;
    sa = s0;
    sb = s1;
}


// Fast path for one star with n <= K vertices and distinct values.  Returns false
// (nothing written) when two star values tie.
// Rank masks of a K-vertex star fit K bits: the per-thread scratch column uses the
// narrowest type (a smaller shared-memory footprint -> more resident blocks).
template <int K>
using MaskT = typename std::conditional<(K <= 8), std::uint8_t,
                                        typename std::conditional<(K <= 16), std::uint16_t, std::uint32_t>::type>::type;

template <int K, typename T, typename Val>
__device__ __forceinline__ bool star_fast(Val val, std::uint32_t S, int n,
                                          const std::uint32_t* fac, const std::uint32_t* cof,
                                          MaskT<K>* mscratch, int mstride, StarWriter& w) {
    using KT = typename KeyOf<T>::type;
    KT key[K];
    std::uint32_t slot[K];
    std::uint32_t rest = S;
#pragma unroll
    for (int p = 0; p < K; ++p) {
        if (p < n) {
            const int s = __ffs(rest) - 1;
            rest &= rest - 1;
            slot[p] = static_cast<std::uint32_t>(s);
            key[p] = ord_key(val(s));
        } else {
            slot[p] = 31u;
            key[p] = static_cast<KT>(~static_cast<KT>(0));
        }
    }
    // (1) vertices by value: Batcher odd-even merge sort with explicit comparator lists
    //     (sortnet.cuh; 19 / 63 / 156 comparators for 8 / 16 / <= 27 vertices, against
    //     24 / 80 / 240 for bitonic networks of 8 / 16 / 32)
    SortNet<(K > 27 ? 27 : K)>::run(
        [&](int a, int b) { ce_pair(key[a], slot[a], key[b], slot[b], true); });
    bool tie = false;
#pragma unroll
    for (int p = 0; p + 1 < K; ++p)
        if (p + 1 < n) tie |= key[p] == key[p + 1];
    if (tie) return false;
    // (2) rank of every star vertex (the centre is the largest: rank n-1)
    Pack5 rank;
#pragma unroll
    for (int p = 0; p < K; ++p)
        if (p < n) rank.set(static_cast<int>(slot[p]), static_cast<std::uint32_t>(p));
    // (3) rank mask of every star cell, from its facets' masks (constant slots)
    std::uint32_t M[27];
#pragma unroll
    for (int t = 0; t < 27; ++t) M[t] = 0;
    M[13] = 1u << (n - 1);
    mscratch[13 * mstride] = static_cast<MaskT<K>>(M[13]);
#pragma unroll
    for (int dim = 1; dim <= 3; ++dim)
#pragma unroll
        for (int t = 0; t < 27; ++t) {
            if (slot_dim(t) != dim) continue;
            std::uint32_t m = 0;
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                const int o = slot_off(t, a);
                if (o != 0) m |= M[t - o * (a == 0 ? 1 : (a == 1 ? 3 : 9))];
            }
            if ((S >> t) & 1u) {
                m |= 1u << rank.get(t);
                mscratch[t * mstride] = static_cast<MaskT<K>>(m);
            }
            M[t] = m;
        }
    // (4) expansion: pop-min = the candidate cell of least rank mask (candidate
    //     sets are small, so a scan over them beats sorting all cells)
    robins(S, fac, cof,
           [&](std::uint32_t m) {
               int best = __ffs(m) - 1;
               if (!(m & (m - 1))) return best;  // a single candidate (the common case)
               std::uint32_t bv = mscratch[best * mstride];
               for (m &= m - 1; m; m &= m - 1) {
                   const int t = __ffs(m) - 1;
                   const std::uint32_t v = mscratch[t * mstride];
                   if (v < bv) {
                       bv = v;
                       best = t;
                   }
               }
               return best;
           },
           w);
    return true;
}

// Octant star (see g_oct): returns false (nothing written) unless S is exactly one
// unit cube at the vertex with 7 distinct link values.  `base` points at the vertex
// in the shared tile.
__device__ __forceinline__ bool is_octant(std::uint32_t S) {
    const std::uint32_t cube = S & kDim3;
    if (__popc(cube) != 1) return false;
    const int c = __ffs(cube) - 1;
    const int sx = (c % 3) - 1, sy = ((c / 3) % 3) - 1, sz = c / 9 - 1;  // each +-1
    return S == ((kX0 | (sx > 0 ? kXP : kXM)) & (kY0 | (sy > 0 ? kYP : kYM)) & (kZ0 | (sz > 0 ? kZP : kZM)));
}

template <typename T>
__device__ __forceinline__ bool octant_fast(const T* base, std::uint32_t S, const std::uint16_t* oct_table,
                                            StarWriter& w) {
    // S is an octant (is_octant): its cube slot gives the orientation
    const int c = __ffs(S & kDim3) - 1;
    const int sx = (c % 3) - 1, sy = ((c / 3) % 3) - 1, sz = c / 9 - 1;  // each +-1
    const int dx = sx, dy = sy * SX, dz = sz * (SX * SY);
    T f[8];
    f[1] = base[dx];
    f[2] = base[dy];
    f[3] = base[dx + dy];
    f[4] = base[dz];
    f[5] = base[dx + dz];
    f[6] = base[dy + dz];
    f[7] = base[dx + dy + dz];
    int idx = 0;
    bool tie = false;
#pragma unroll
    for (int i = 1; i <= 7; ++i) {
        int below = 0;
#pragma unroll
        for (int j = i + 1; j <= 7; ++j) {
            below += f[j] < f[i];
            tie |= f[j] == f[i];
        }
        constexpr int kFact[8] = {0, 720, 120, 24, 6, 2, 1, 1};
        idx += below * kFact[i];
    }
    if (tie) return false;
    const std::uint32_t e = __ldg(&oct_table[idx]);
    const int st[3] = {sx, 3 * sy, 9 * sz};
#pragma unroll
    for (int m = 1; m < 8; ++m) {
        const int a = static_cast<int>((e >> (2 * m)) & 3u);
        const int sm = 13 + (m & 1) * st[0] + ((m >> 1) & 1) * st[1] + ((m >> 2) & 1) * st[2];
        if (a == 0) {
            w.critical(sm, __popc(m));
        } else if ((m >> (a - 1)) & 1) {  // the higher cell of the pair writes it
            const int lo = m ^ (1 << (a - 1));
            w.pair(13 + (lo & 1) * st[0] + ((lo >> 1) & 1) * st[1] + ((lo >> 2) & 1) * st[2], sm);
        }
    }
    return true;
}

// Work lists handed from the tile kernel to the size-specialised kernels:
// [0] stars of 9..16 cells, [1] 17..27 cells, [2] stars with tied values.
struct StarLists {
    std::uint32_t* list[3];
    std::uint32_t* mask[2];     // lists 0/1: the star's slot mask S, computed by the tile kernel
    unsigned long long* count;  // 3 counters, then 3 chunk heads for the list kernels
};

// Block-level buffers for the large-star work lists: appends are shared-memory
// atomics; the global list counters are touched once per flush (a counter hit by
// every thread of the grid serialises in the L2).
constexpr int kListBuf = 1024;

// ---- TMA tile loads (sm_90+ tensor memory accelerator; Blackwell sm_100a) -------------
// One elected thread issues the box copy global -> shared for each tile of a group;
// completion is tracked by a transaction-count mbarrier per buffer set, which every
// thread waits on (parity) before reading the tile.  Out-of-box coordinates (the -1
// halo, tiles past the grid) are zero-filled by the hardware, as the cp.async path
// does by hand.
__device__ __forceinline__ void mbar_init(std::uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(bar))),
                 "r"(count)
                 : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(std::uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                     static_cast<unsigned>(__cvta_generic_to_shared(bar))),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(std::uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(bar))),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z,
                                            std::uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
            "r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))),
        "l"(reinterpret_cast<std::uint64_t>(map)), "r"(x), "r"(y), "r"(z),
        "r"(static_cast<unsigned>(__cvta_generic_to_shared(bar)))
        : "memory");
}

template <typename T, bool kTma>
__global__ void __launch_bounds__(NT, 5)
k_gradient(const T* __restrict__ f, Dims d, std::uint8_t* __restrict__ codes,
           std::uint32_t* __restrict__ parent0, std::uint32_t* __restrict__ parent3,
           unsigned long long* __restrict__ crit_totals, StarLists lists, uint3 tiles, unsigned tz_first,
           const __grid_constant__ CUtensorMap tmap) {
    // Tiles go in groups of kGroup (consecutive along x): phase 1 bins the group's
    // 3..8-cell stars by size, phase 2 runs them all -- ~2x the work per barrier, so
    // fewer idle lanes.  f32: two buffer sets, the next group streams in (cp.async)
    // while this one is processed; f64: one set (static shared memory budget).
    constexpr int kGroup = 2;
    constexpr int kSets = sizeof(T) == 4 ? 2 : 1;
    __shared__ alignas(128) T tiles_sm[kSets][kGroup][SZ][SY][SX];
    __shared__ alignas(8) std::uint64_t s_bar[kSets];  // TMA: one transaction barrier per buffer set
    __shared__ std::uint32_t s_fac[27], s_cof[27];
    __shared__ std::int32_t s_cell[27];
    __shared__ std::uint32_t s_coff[27];
    __shared__ unsigned long long s_crit[4];
    __shared__ MaskT<8> s_M[27 * NT];
    __shared__ std::uint32_t s_lb[2][kListBuf];
    __shared__ std::uint32_t s_lm[2][kListBuf];
    __shared__ std::uint32_t s_ln[2];
    __shared__ unsigned long long s_base[2];
    // phase-2 work list: buckets of star size 3..8, then unit-cube (octant) stars
    __shared__ std::uint32_t s_wn[7], s_wtotal, s_woct;
    __shared__ std::uint32_t s_wS[kGroup * NT];
    __shared__ std::uint16_t s_wid[kGroup * NT];  // tile-in-group << 8 | vertex in tile
    const int tid = threadIdx.x + TX * (threadIdx.y + TY * threadIdx.z);
    // the tensor map stays in the kernel's parameter space (a copy in local memory is
    // not a valid TMA operand): its address is taken here, outside the lambdas
    const CUtensorMap* tmap_p = &tmap;
    if (tid < 27) {
        s_fac[tid] = c_slot.facet[tid];
        s_cof[tid] = c_slot.cofacet[tid];
        s_coff[tid] = cube_slot_offset(tid, d);
        s_cell[tid] = static_cast<std::int32_t>(c_slot.off[tid][0] + c_slot.off[tid][1] * d.ex +
                                                c_slot.off[tid][2] * d.exy);
    }
    if (tid < 4) s_crit[tid] = 0;
    if (tid < 2) s_ln[tid] = 0;
    auto flush_lists = [&]() {  // all threads
        __syncthreads();
        if (tid < 2) s_base[tid] = s_ln[tid] ? atomicAdd(&lists.count[tid], static_cast<unsigned long long>(s_ln[tid])) : 0ull;
        __syncthreads();
#pragma unroll
        for (int w = 0; w < 2; ++w)
            for (std::uint32_t k = tid; k < s_ln[w]; k += NT) {
                lists.list[w][s_base[w] + k] = s_lb[w][k];
                lists.mask[w][s_base[w] + k] = s_lm[w][k];
            }
        __syncthreads();
        if (tid < 2) s_ln[tid] = 0;
        __syncthreads();
    };
    std::uint32_t crit[4] = {0, 0, 0, 0};
    const std::uint64_t ntiles = static_cast<std::uint64_t>(tiles.x) * tiles.y * tiles.z;
    const std::uint64_t ngroups = (ntiles + kGroup - 1) / kGroup;
    // tile origin (shared-memory column 0 = x - XO; the -1 halo corner in y and z),
    // 32-bit: tile ids and coordinates fit
    auto origin = [&](std::uint64_t ti, std::int64_t& x0, std::int64_t& y0, std::int64_t& z0) {
        const std::uint32_t t32 = static_cast<std::uint32_t>(ti);
        const std::uint32_t tyz = t32 / tiles.x;
        x0 = static_cast<std::int64_t>(static_cast<int>((t32 - tyz * tiles.x) * TX) - XO);
        y0 = static_cast<std::int64_t>(static_cast<int>((tyz % tiles.y) * TY) - 1);
        z0 = static_cast<std::int64_t>(static_cast<int>((tyz / tiles.y + tz_first) * TZ) - 1);
    };
    // element offsets inside a tile fit 32 bits when a 4-plane slab does
    const bool off32 = static_cast<std::uint64_t>(d.nx) * d.ny * SZ < (1ull << 31);
    const int nx32 = static_cast<int>(d.nx), nxy32 = static_cast<int>(d.nx * d.ny);
    // group gi's tiles (+1 halo) -> buffer set b: in-range samples by asynchronous
    // copies, the rest (and tiles past the end) 0.  Interior tiles (the common case)
    // skip the per-sample range checks.
    auto load_group = [&](std::uint64_t gi, int b) {
        if constexpr (kTma) {
            if (tid == 0) {
                // the generic-proxy reads of this buffer set are done (barrier before)
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_expect_tx(&s_bar[b], kGroup * kTileBytesF32);
                for (int g = 0; g < kGroup; ++g) {
                    std::int64_t x0, y0, z0;
                    origin(gi * kGroup + g, x0, y0, z0);  // past the last tile: z0 >= nz, all zero-filled
                    tma_load_3d(&tiles_sm[b][g][0][0][0], tmap_p, static_cast<int>(x0), static_cast<int>(y0),
                                static_cast<int>(z0), &s_bar[b]);
                }
            }
            return;
        }
        for (int g = 0; g < kGroup; ++g) {
            const std::uint64_t ti = gi * kGroup + g;
            std::int64_t x0, y0, z0;
            origin(ti, x0, y0, z0);
            T* dst = &tiles_sm[b][g][0][0][0];
            const bool interior = off32 && ti < ntiles && x0 >= 0 && x0 + SX <= d.nx && y0 >= 0 && y0 + SY <= d.ny &&
                                  z0 >= 0 && z0 + SZ <= d.nz;
            if (interior) {
                const T* fb = f + (x0 + d.nx * (y0 + d.ny * z0));
                for (int i = tid; i < SX * SY * SZ; i += NT) {
                    const int lz = i / (SX * SY), r = i - lz * (SX * SY), ly = r / SX, lx = r - ly * SX;
                    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(dst + i));
                    const T* src = fb + (lx + nx32 * ly + nxy32 * lz);
                    if (sizeof(T) == 4)
                        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(src) : "memory");
                    else
                        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(src) : "memory");
                }
                continue;
            }
            for (int i = tid; i < SX * SY * SZ; i += NT) {
                const int lz = i / (SX * SY), r = i - lz * (SX * SY), ly = r / SX, lx = r - ly * SX;
                const std::int64_t gx = x0 + lx, gy = y0 + ly, gz = z0 + lz;
                if (ti < ntiles && gx >= 0 && gx < d.nx && gy >= 0 && gy < d.ny && gz >= 0 && gz < d.nz) {
                    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(dst + i));
                    const T* src = f + gx + d.nx * (gy + d.ny * gz);
                    if (sizeof(T) == 4)
                        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(src) : "memory");
                    else
                        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(src) : "memory");
                } else {
                    dst[i] = T(0);
                }
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    unsigned phase = 0;  // TMA: parity bit of each set's barrier (bit b)
    if constexpr (kTma) {
        if (tid == 0) {
            for (int b = 0; b < kSets; ++b) mbar_init(&s_bar[b], 1);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the barriers, visible to the TMA unit
        }
        __syncthreads();
    }
    if (blockIdx.x < ngroups) load_group(blockIdx.x, 0);
    int cur = 0;
    for (std::uint64_t gi = blockIdx.x; gi < ngroups; gi += gridDim.x) {
        if constexpr (kTma) {
            mbar_wait(&s_bar[cur], (phase >> cur) & 1u);
            phase ^= 1u << cur;
        } else {
            asm volatile("cp.async.wait_all;" ::: "memory");
        }
        __syncthreads();  // group gi in shared memory; the previous group's work done
        if (s_ln[0] + kGroup * NT > kListBuf || s_ln[1] + kGroup * NT > kListBuf) flush_lists();
        const std::uint64_t gn = gi + gridDim.x;
        if (kSets == 2 && gn < ngroups) load_group(gn, cur ^ 1);  // overlaps this group's work
        const int set = cur;
        if (kSets == 2) cur ^= 1;

        // this group's tile origins, once (kGroup == 2: selects, not indexed arrays)
        static_assert(kGroup == 2, "origins below are written out for pairs of tiles");
        std::int64_t ox0, oy0, oz0, ox1, oy1, oz1;
        origin(gi * kGroup, ox0, oy0, oz0);
        origin(gi * kGroup + 1, ox1, oy1, oz1);
        auto writer_for = [&](int g, int lid, StarWriter& w) {  // false: vertex outside the grid
            const std::uint64_t ti = gi * kGroup + g;
            if (ti >= ntiles) return false;
            const std::int64_t x0 = g ? ox1 : ox0, y0 = g ? oy1 : oy0, z0 = g ? oz1 : oz0;
            const int lx = lid % TX, ly = (lid / TX) % TY, lz = lid / (TX * TY);
            w.vx = x0 + XO + lx;
            w.vy = y0 + 1 + ly;
            w.vz = z0 + 1 + lz;
            if (w.vx >= d.nx || w.vy >= d.ny || w.vz >= d.nz) return false;
            std::uint32_t inr = kAll;
            if (w.vx == 0) inr &= ~kXM;
            if (w.vx == d.nx - 1) inr &= ~kXP;
            if (w.vy == 0) inr &= ~kYM;
            if (w.vy == d.ny - 1) inr &= ~kYP;
            if (w.vz == 0) inr &= ~kZM;
            if (w.vz == d.nz - 1) inr &= ~kZP;
            w.inr = inr;
            w.d = d;
            w.cbase = codes + (2 * w.vx + d.ex * (2 * w.vy + d.ey * 2 * w.vz));
            w.cell_off = s_cell;
            w.cube_off = s_coff;
            w.parent0 = parent0;
            w.parent3 = parent3;
            w.ncrit = 0;
            w.init_cubes();
            return true;
        };
        // ---- phase 1, own vertex of each tile: star mask; trivial stars finished here;
        //      stars of 3..8 cells binned by size; larger stars to the list kernels
        if (tid < 7) s_wn[tid] = 0;
        __syncthreads();
        int ng[kGroup];
        std::uint32_t Sg[kGroup];
#pragma unroll
        for (int g = 0; g < kGroup; ++g) {
            ng[g] = 0;
            Sg[g] = 0;
            StarWriter w;
            if (writer_for(g, tid, w)) {
                const T* base = &tiles_sm[set][g][threadIdx.z + 1][threadIdx.y + 1][threadIdx.x + XO];
                const T fv = base[0];
                std::uint32_t below = kCentre;
#pragma unroll
                for (int t = 0; t < 27; ++t) {
                    if (t == 13) continue;
                    const T u = base[slot_tile(t)];
                    if (u < fv || (u == fv && t < 13)) below |= 1u << t;
                }
                std::uint32_t S = below & w.inr;
                S &= facets_present(S);
                S &= facets_present(S);
                const int n = __popc(S);
                if (n == 1) {  // critical minimum (gradient.cpp:128-131)
                    w.minimum();
                } else if (n == 2) {  // the vertex and its only edge pair up
                    w.pair(13, __ffs(S & ~kCentre) - 1);
                } else if (n > 8) {
                    const int which = n <= 16 ? 0 : 1;
                    const std::uint32_t at = atomicAdd(&s_ln[which], 1u);
                    s_lb[which][at] = static_cast<std::uint32_t>(w.vx + d.nx * (w.vy + d.ny * w.vz));
                    s_lm[which][at] = S;
                } else {
                    const int bucket = (n == 8 && is_octant(S)) ? 6 : n - 3;
                    atomicAdd(&s_wn[bucket], 1u);
                    ng[g] = bucket + 3;
                    Sg[g] = S;
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) crit[k] += static_cast<std::uint32_t>((w.ncrit >> (16 * k)) & 0xffffu);
            }
        }
        __syncthreads();
        if (tid == 0) {
            std::uint32_t acc = 0;
            for (int k = 0; k < 7; ++k) {
                const std::uint32_t c = s_wn[k];
                s_wn[k] = acc;
                acc += c;
            }
            s_wtotal = acc;
            s_woct = s_wn[6];
        }
        __syncthreads();
#pragma unroll
        for (int g = 0; g < kGroup; ++g)
            if (ng[g] >= 3) {
                const std::uint32_t at = atomicAdd(&s_wn[ng[g] - 3], 1u);
                s_wS[at] = Sg[g];
                s_wid[at] = static_cast<std::uint16_t>((g << 8) | tid);
            }
        __syncthreads();
        // the table path pays off where unit-cube stars dominate (smooth fields); on
        // noisy tiles the generic path is as fast and the two would diverge
        const bool use_oct = 4 * (s_wtotal - s_woct) >= 3 * s_wtotal;
        // ---- phase 2: the binned stars, one per thread, register fast path
        for (std::uint32_t k = tid; k < s_wtotal; k += NT) {
            const int g = s_wid[k] >> 8, lid = s_wid[k] & 0xff;
            const std::uint32_t Sw = s_wS[k];
            StarWriter w;
            writer_for(g, lid, w);
            const T* base = &tiles_sm[set][g][lid / (TX * TY) + 1][(lid / TX) % TY + 1][lid % TX + XO];
            if (use_oct && k >= s_woct && octant_fast<T>(base, Sw, g_oct, w)) {
                // a unit-cube star: paired from the table (false only on tied values)
            } else if (!star_fast<8, T>([&](int t) { return base[tile_off(t)]; }, Sw, __popc(Sw), s_fac, s_cof,
                                        &s_M[tid], NT, w)) {
                const unsigned long long at = atomicAdd(&lists.count[2], 1ull);  // ties: rare
                lists.list[2][at] = static_cast<std::uint32_t>(w.vx + d.nx * (w.vy + d.ny * w.vz));
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) crit[q] += static_cast<std::uint32_t>((w.ncrit >> (16 * q)) & 0xffffu);
        }
        if (kSets == 1 && gn < ngroups) {
            __syncthreads();  // everyone done with the single buffer set
            load_group(gn, 0);
        }
    }
    flush_lists();
    if (crit_totals) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            std::uint32_t v = crit[k];
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if ((tid & 31) == 0 && v) atomicAdd(&s_crit[k], static_cast<unsigned long long>(v));
        }
        __syncthreads();
        if (tid < 4 && s_crit[tid]) atomicAdd(&crit_totals[tid], s_crit[tid]);
    }
}

// Stars of 9..27 cells, one thread per listed vertex (values from global memory,
// L1/L2-resident neighbourhoods).  Same register fast path with a wider network;
// tied stars are forwarded to the slow path list.
template <int K, typename T>
__global__ void __launch_bounds__(128, K == 32 ? 7 : 8)
k_gradient_list(const T* __restrict__ f, Dims d, std::uint8_t* __restrict__ codes,
                std::uint32_t* __restrict__ parent0, std::uint32_t* __restrict__ parent3,
                unsigned long long* __restrict__ crit_totals, StarLists lists, int which) {
    __shared__ std::int32_t s_cell[27];
    __shared__ std::uint32_t s_coff[27];
    __shared__ std::uint32_t s_fac[27], s_cof[27];
    __shared__ MaskT<K> s_M[27 * 128];
    __shared__ unsigned long long s_crit[4];
    __shared__ long long s_voff[27];  // sample offset of slot t from the star's vertex
    if (threadIdx.x < 27) {
        s_fac[threadIdx.x] = c_slot.facet[threadIdx.x];
        s_cof[threadIdx.x] = c_slot.cofacet[threadIdx.x];
        s_coff[threadIdx.x] = cube_slot_offset(static_cast<int>(threadIdx.x), d);
        s_cell[threadIdx.x] = static_cast<std::int32_t>(
            c_slot.off[threadIdx.x][0] + c_slot.off[threadIdx.x][1] * d.ex + c_slot.off[threadIdx.x][2] * d.exy);
        s_voff[threadIdx.x] = c_slot.off[threadIdx.x][0] + c_slot.off[threadIdx.x][1] * d.nx +
                              c_slot.off[threadIdx.x][2] * d.nx * d.ny;
    }
    if (threadIdx.x < 4) s_crit[threadIdx.x] = 0;
    __syncthreads();
    const std::uint64_t nl = *reinterpret_cast<volatile unsigned long long*>(&lists.count[which]);
    std::uint64_t ncrit = 0;
    // chunks of blockDim.x list entries taken in list (= spatial) order by whichever
    // block is free: the grid sweeps the volume as one wavefront
    __shared__ unsigned long long s_chunk;
    for (;;) {
        __syncthreads();
        if (threadIdx.x == 0) s_chunk = atomicAdd(&lists.count[3 + which], 1ull);
        __syncthreads();
        const std::uint64_t i = s_chunk * blockDim.x + threadIdx.x;
        if (s_chunk * blockDim.x >= nl) break;
        if (i >= nl) continue;
        const std::uint32_t vi = lists.list[which][i];
        const std::uint64_t r = d.fnx.div(vi), vx = vi - r * d.nx, vz = d.fny.div(r), vy = r - vz * d.ny;
        StarWriter w;
        w.vx = static_cast<std::int64_t>(vx);
        w.vy = static_cast<std::int64_t>(vy);
        w.vz = static_cast<std::int64_t>(vz);
        std::uint32_t inr = kAll;
        if (w.vx == 0) inr &= ~kXM;
        if (w.vx == d.nx - 1) inr &= ~kXP;
        if (w.vy == 0) inr &= ~kYM;
        if (w.vy == d.ny - 1) inr &= ~kYP;
        if (w.vz == 0) inr &= ~kZM;
        if (w.vz == d.nz - 1) inr &= ~kZP;
        w.inr = inr;
        w.d = d;
        w.cbase = codes + (2 * w.vx + d.ex * (2 * w.vy + d.ey * 2 * w.vz));
        w.cell_off = s_cell;
        w.cube_off = s_coff;
        w.parent0 = parent0;
        w.parent3 = parent3;
        w.ncrit = 0;
        w.init_cubes();
        const T* centre = f + vi;
        const std::int64_t sy = d.nx, sz = d.nx * d.ny;
        auto val = [&](int t) { return centre[s_voff[t]]; };
        std::uint32_t S;
        if (K == 16) {
            S = lists.mask[which][i];  // from the tile kernel
        } else {  // (recomputing it measured faster here: fewer live registers across the loads)
            const T fv = centre[0];
            std::uint32_t below = kCentre;
#pragma unroll
            for (int t = 0; t < 27; ++t) {
                if (t == 13) continue;
                if (!((inr >> t) & 1u)) continue;
                const T u = centre[slot_off(t, 0) + slot_off(t, 1) * sy + slot_off(t, 2) * sz];
                if (u < fv || (u == fv && t < 13)) below |= 1u << t;
            }
            S = below & inr;
            S &= facets_present(S);
            S &= facets_present(S);
        }
        if (!star_fast<K, T>(val, S, __popc(S), s_fac, s_cof, &s_M[threadIdx.x], 128, w)) {
            const unsigned long long at = atomicAdd(&lists.count[2], 1ull);
            lists.list[2][at] = vi;
        }
        ncrit += w.ncrit;
    }
    std::uint64_t v = ncrit;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0 && v)
        for (int k = 0; k < 4; ++k) {
            const unsigned long long c = (v >> (16 * k)) & 0xffffu;
            if (c) atomicAdd(&s_crit[k], c);
        }
    __syncthreads();
    if (threadIdx.x < 4 && s_crit[threadIdx.x]) atomicAdd(&crit_totals[threadIdx.x], s_crit[threadIdx.x]);
}

// Slow path: stars with equal values.  The general key of the reference
// (value multiset, then vertex ids), one thread per deferred vertex, values read
// straight from global memory.
template <typename T>
__global__ void __launch_bounds__(128)
k_gradient_deferred(const T* __restrict__ f, Dims d, std::uint8_t* __restrict__ codes,
                    std::uint32_t* __restrict__ parent0, std::uint32_t* __restrict__ parent3,
                    StarLists lists, unsigned long long* __restrict__ crit_totals) {
    __shared__ std::int32_t s_cell[27];
    __shared__ std::uint32_t s_coff[27];
    __shared__ std::uint32_t s_fac[27], s_cof[27];
    if (threadIdx.x < 27) {
        s_fac[threadIdx.x] = c_slot.facet[threadIdx.x];
        s_cof[threadIdx.x] = c_slot.cofacet[threadIdx.x];
        s_coff[threadIdx.x] = cube_slot_offset(static_cast<int>(threadIdx.x), d);
        s_cell[threadIdx.x] = static_cast<std::int32_t>(
            c_slot.off[threadIdx.x][0] + c_slot.off[threadIdx.x][1] * d.ex + c_slot.off[threadIdx.x][2] * d.exy);
    }
    __syncthreads();
    const std::uint64_t nl = *reinterpret_cast<volatile unsigned long long*>(&lists.count[2]);
    for (std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x; i < nl;
         i += static_cast<std::uint64_t>(gridDim.x) * blockDim.x) {
        const std::uint32_t vi = lists.list[2][i];
        const std::uint64_t r = d.fnx.div(vi), vx = vi - r * d.nx, vz = d.fny.div(r), vy = r - vz * d.ny;
        StarWriter w;
        w.vx = static_cast<std::int64_t>(vx);
        w.vy = static_cast<std::int64_t>(vy);
        w.vz = static_cast<std::int64_t>(vz);
        std::uint32_t inr = kAll;
        if (w.vx == 0) inr &= ~kXM;
        if (w.vx == d.nx - 1) inr &= ~kXP;
        if (w.vy == 0) inr &= ~kYM;
        if (w.vy == d.ny - 1) inr &= ~kYP;
        if (w.vz == 0) inr &= ~kZM;
        if (w.vz == d.nz - 1) inr &= ~kZP;
        w.inr = inr;
        w.d = d;
        w.cbase = codes + (2 * w.vx + d.ex * (2 * w.vy + d.ey * 2 * w.vz));
        w.cell_off = s_cell;
        w.cube_off = s_coff;
        w.parent0 = parent0;
        w.parent3 = parent3;
        w.ncrit = 0;
        w.init_cubes();
        auto val = [&](int t) {
            const std::int64_t ox = t % 3 - 1, oy = (t / 3) % 3 - 1, oz = t / 9 - 1;
            return f[(w.vx + ox) + d.nx * ((w.vy + oy) + d.ny * (w.vz + oz))];
        };
        const T fv = val(13);
        std::uint32_t below = kCentre;
        for (int t = 0; t < 27; ++t) {
            if (t == 13 || !((inr >> t) & 1u)) continue;
            const T u = val(t);
            if (u < fv || (u == fv && t < 13)) below |= 1u << t;
        }
        std::uint32_t S = below & inr;
        S &= facets_present(S);
        S &= facets_present(S);
        // top rank of each star vertex's equal-value group, then the general key
        std::uint8_t top[27];
        for (std::uint32_t m = S; m; m &= m - 1) {
            const int s = __ffs(m) - 1;
            const T vs = val(s);
            int c = -1;
            for (std::uint32_t q = S; q; q &= q - 1) c += val(__ffs(q) - 1) <= vs;
            top[s] = static_cast<std::uint8_t>(c);
        }
        std::uint64_t key[27];
        for (std::uint32_t m = S & ~kCentre; m; m &= m - 1) {
            const int t = __ffs(m) - 1;
            std::uint32_t vm = 0;
            for (std::uint32_t q = c_slot.sub[t]; q; q &= q - 1) {
                int b = top[__ffs(q) - 1];
                while ((vm >> b) & 1u) --b;
                vm |= 1u << b;
            }
            key[t] = (static_cast<std::uint64_t>(vm) << 27) | c_slot.sub[t];
        }
        robins(S, s_fac, s_cof,
               [&](std::uint32_t m) {
                   int best = __ffs(m) - 1;
                   std::uint64_t bk = key[best];
                   for (m &= m - 1; m; m &= m - 1) {
                       const int t = __ffs(m) - 1;
                       if (key[t] < bk) {
                           bk = key[t];
                           best = t;
                       }
                   }
                   return best;
               },
               w);
        if (crit_totals)
            for (int k = 0; k < 4; ++k) {
                const unsigned long long c = (w.ncrit >> (16 * k)) & 0xffffu;
                if (c) atomicAdd(&crit_totals[k], c);
            }
    }
}

bool g_tables_ready[64] = {false};

// The samples as a 3-D tensor (x fastest) with a 36 x 6 x 4 box: one TMA copy per tile.
// Needs 16-byte row strides (nx % 4 == 0) and an aligned base; false -> the cp.async path.
// cuTensorMapEncodeTiled comes from the driver through the runtime's entry-point query,
// so the library does not link libcuda.
bool f32_tensor_map(const void* values, const Dims& d, CUtensorMap* map) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    static bool tried = false;
    if (std::getenv("MSC3D_NO_TMA")) return false;
    if (!tried) {
        tried = true;
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
        else
            cudaGetLastError();
    }
    if (!encode || d.nx % 4 != 0 || (reinterpret_cast<std::uintptr_t>(values) & 15) != 0) return false;
    const cuuint64_t dims[3] = {static_cast<cuuint64_t>(d.nx), static_cast<cuuint64_t>(d.ny),
                                static_cast<cuuint64_t>(d.nz)};
    const cuuint64_t strides[2] = {static_cast<cuuint64_t>(d.nx) * 4, static_cast<cuuint64_t>(d.nx * d.ny) * 4};
    const cuuint32_t box[3] = {SX, SY, SZ};
    const cuuint32_t estr[3] = {1, 1, 1};
    return encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(values), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

int upload_gradient_tables(int device) {
    if (device >= 0 && device < 64 && g_tables_ready[device]) return MSC3D_OK;
    const SlotTables t = host_tables();
    MSC3D_CUDA_TRY(cudaMemcpyToSymbol(c_slot, &t, sizeof t));
    const std::vector<std::uint16_t> oct = host_octant_table();
    MSC3D_CUDA_TRY(cudaMemcpyToSymbol(g_oct, oct.data(), oct.size() * sizeof(std::uint16_t)));
    if (device >= 0 && device < 64) g_tables_ready[device] = true;
    return MSC3D_OK;
}

int gradient_begin(unsigned long long* crit_totals, unsigned long long* list_counts, cudaStream_t stream) {
    int dev = 0;
    MSC3D_CUDA_TRY(cudaGetDevice(&dev));
    const int rc = upload_gradient_tables(dev);
    if (rc != MSC3D_OK) return rc;
    MSC3D_CUDA_TRY(cudaMemsetAsync(crit_totals, 0, 32, stream));
    MSC3D_CUDA_TRY(cudaMemsetAsync(list_counts, 0, 48, stream));
    return MSC3D_OK;
}

unsigned gradient_tile_layers(const Dims& d) { return static_cast<unsigned>((d.nz + TZ - 1) / TZ); }
int gradient_layer_last_plane(const Dims& d, unsigned tz_end) {  // last vertex plane the layers read
    return static_cast<int>(std::min<std::int64_t>(d.nz - 1, static_cast<std::int64_t>(tz_end) * TZ));
}

int gradient_tiles(const void* values, int value_type, const Dims& d, std::uint8_t* codes, std::uint32_t* parent0,
                   std::uint32_t* parent3, cudaStream_t stream, unsigned long long* crit_totals,
                   std::uint32_t* const lists3[3], unsigned long long* list_counts, int num_sms, unsigned tz0,
                   unsigned tz1) {
    if (tz1 <= tz0) return MSC3D_OK;
    // lists 0/1 hold 2 * n_verts entries: ids, then the stars' slot masks
    StarLists lists{{lists3[0], lists3[1], lists3[2]}, {lists3[0] + d.n_verts, lists3[1] + d.n_verts}, list_counts};
    const dim3 block(TX, TY, TZ);
    const uint3 tiles = make_uint3(static_cast<unsigned>((d.nx + TX - 1) / TX),
                                   static_cast<unsigned>((d.ny + TY - 1) / TY), tz1 - tz0);
    const std::uint64_t ntiles = static_cast<std::uint64_t>(tiles.x) * tiles.y * tiles.z;
    // persistent tile loop: a few blocks per SM, each walking tiles with stride grid
    const dim3 grid(static_cast<unsigned>(std::min<std::uint64_t>(ntiles, static_cast<std::uint64_t>(num_sms) * 8)));
    CUtensorMap tmap;
    if (value_type == MSC3D_VALUE_F64)
        k_gradient<double, false><<<grid, block, 0, stream>>>(static_cast<const double*>(values), d, codes, parent0,
                                                              parent3, crit_totals, lists, tiles, tz0, tmap);
    else if (f32_tensor_map(values, d, &tmap))
        k_gradient<float, true><<<grid, block, 0, stream>>>(static_cast<const float*>(values), d, codes, parent0,
                                                            parent3, crit_totals, lists, tiles, tz0, tmap);
    else
        k_gradient<float, false><<<grid, block, 0, stream>>>(static_cast<const float*>(values), d, codes, parent0,
                                                             parent3, crit_totals, lists, tiles, tz0, tmap);
    count_launch();
    MSC3D_CUDA_TRY(cudaGetLastError());
    return MSC3D_OK;
}

int gradient_finish(const void* values, int value_type, const Dims& d, std::uint8_t* codes, std::uint32_t* parent0,
                    std::uint32_t* parent3, cudaStream_t stream, unsigned long long* crit_totals,
                    std::uint32_t* const lists3[3], unsigned long long* list_counts, int num_sms) {
    // lists 0/1 hold 2 * n_verts entries: ids, then the stars' slot masks
    StarLists lists{{lists3[0], lists3[1], lists3[2]}, {lists3[0] + d.n_verts, lists3[1] + d.n_verts}, list_counts};
    const unsigned lgrid = static_cast<unsigned>(16 * num_sms);
    const unsigned dgrid = static_cast<unsigned>(4 * num_sms);
    if (value_type == MSC3D_VALUE_F64) {
        const double* v = static_cast<const double*>(values);
        k_gradient_list<16, double><<<lgrid, 128, 0, stream>>>(v, d, codes, parent0, parent3, crit_totals, lists, 0);
        k_gradient_list<32, double><<<lgrid, 128, 0, stream>>>(v, d, codes, parent0, parent3, crit_totals, lists, 1);
        k_gradient_deferred<double><<<dgrid, 128, 0, stream>>>(v, d, codes, parent0, parent3, lists, crit_totals);
    } else {
        const float* v = static_cast<const float*>(values);
        k_gradient_list<16, float><<<lgrid, 128, 0, stream>>>(v, d, codes, parent0, parent3, crit_totals, lists, 0);
        k_gradient_list<32, float><<<lgrid, 128, 0, stream>>>(v, d, codes, parent0, parent3, crit_totals, lists, 1);
        k_gradient_deferred<float><<<dgrid, 128, 0, stream>>>(v, d, codes, parent0, parent3, lists, crit_totals);
    }
    count_launch(3);
    MSC3D_CUDA_TRY(cudaGetLastError());
    return MSC3D_OK;
}

int launch_gradient(const void* values, int value_type, const Dims& d, std::uint8_t* codes,
                    std::uint32_t* parent0, std::uint32_t* parent3, cudaStream_t stream,
                    unsigned long long* crit_totals, std::uint32_t* const lists3[3],
                    unsigned long long* list_counts, int num_sms) {
    int rc = gradient_begin(crit_totals, list_counts, stream);
    if (rc == MSC3D_OK)
        rc = gradient_tiles(values, value_type, d, codes, parent0, parent3, stream, crit_totals, lists3, list_counts,
                            num_sms, 0, gradient_tile_layers(d));
    if (rc == MSC3D_OK)
        rc = gradient_finish(values, value_type, d, codes, parent0, parent3, stream, crit_totals, lists3, list_counts,
                             num_sms);
    return rc;
}

}  // namespace msc3d_dev

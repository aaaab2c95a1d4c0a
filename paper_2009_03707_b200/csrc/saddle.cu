// Saddle-saddle stages: DAG successors, reachability, branch contraction and
// 2-saddle-keyed path counting (proj/src/saddle_graph.cpp, proj/src/path_matrix.cpp),
// re-designed for the device.
//
// Node space.  DAG nodes are 1-cells; every per-node array is indexed by the "dense
// edge" index de = 3 * (lower vertex) + axis, so a warp walking consecutive nodes
// touches neighbouring lattice cells (no node renumbering, no id map).  Visited
// nodes are one bit each (3V bits: 50 MB at 512^3, L2-resident).
//
// Successors (saddle_graph.cpp:10-24): for each cofacet quad q of e in cofacet
// order: q critical -> terminal 2-saddle q; q paired with a facet edge e' != e ->
// edge e'; q paired with a cube -> nothing.  Recomputed from the pair codes
// whenever needed (4 byte loads, spatially local) instead of stored.
//
// Reachability (saddle_graph.cpp:26-86): one persistent cooperative kernel runs all
// BFS levels, with a grid barrier per level, warp-aggregated frontier appends and
// an atomic test-and-set per claimed node bit.  The claimed SET equals the
// reference's serial claim-order result.
//
// Counting.  The reference contracts junction-free traces into a minor and then
// multiplies sparse matrices, A* = A(I + B + B^2 ...), A*B* + D.  Here every
// junction / 1-saddle branch is walked to its end (2-saddle, junction or dead end;
// total walk length ~ the node count: 240.6 M trace steps for 243 M
// nodes at config 3), and each junction's sparse vector P(j) of path counts to
// 2-saddles is built in reverse topological order (Kahn's algorithm on the junction
// graph: one persistent kernel, one grid barrier per level) by merging the
// vectors of its branch destinations.  1-saddles merge the same way straight into
// the sorted output.  Counts are exact u64; any overflow is sticky and reported.
#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace msc3d_dev {

namespace {

constexpr int kThreads = 256;
constexpr std::uint32_t kTerm = 0x80000000u;
constexpr std::uint32_t kNone = 0xffffffffu;

// One item per thread (the grid-stride loops below then run once): blocks are
// scheduled in id order, so the resident ones sweep the id space as a compact
// wavefront and spatially neighbouring items share the L2.
inline unsigned grid_for(std::uint64_t n, int /*num_sms*/, int /*per_sm*/ = 16) {
    return static_cast<unsigned>(std::max<std::uint64_t>(1, (n + kThreads - 1) / kThreads));
}

#define GRID_STRIDE(i, n)                                                                       \
    for (std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x; \
         i < (n); i += static_cast<std::uint64_t>(gridDim.x) * blockDim.x)

struct C3 {
    std::int32_t x, y, z;
};

__device__ __forceinline__ std::int64_t cell_id(const Dims& d, const C3& c) {
    return c.x + d.ex * (c.y + d.ey * static_cast<std::int64_t>(c.z));
}
__device__ __forceinline__ std::uint32_t edge_dense(const Dims& d, const C3& c) {
    const int axis = (c.x & 1) ? 0 : ((c.y & 1) ? 1 : 2);
    return 3u * static_cast<std::uint32_t>((c.x >> 1) + d.nx * ((c.y >> 1) + d.ny * (c.z >> 1))) + axis;
}
__device__ __forceinline__ std::uint32_t quad_dense(const Dims& d, const C3& c) {
    const int axis = !(c.x & 1) ? 0 : (!(c.y & 1) ? 1 : 2);
    return 3u * static_cast<std::uint32_t>((c.x >> 1) + d.nx * ((c.y >> 1) + d.ny * (c.z >> 1))) + axis;
}
__device__ __forceinline__ C3 edge_coord(const Dims& d, std::uint32_t de) {
    const std::uint32_t v = __umulhi(de, 0xAAAAAAABu) >> 1, a = de - 3 * v;
    const std::uint64_t r = d.fnx.div(v), vx = v - r * d.nx, vz = d.fny.div(r), vy = r - vz * d.ny;
    C3 c;
    c.x = static_cast<std::int32_t>(2 * vx + (a == 0));
    c.y = static_cast<std::int32_t>(2 * vy + (a == 1));
    c.z = static_cast<std::int32_t>(2 * vz + (a == 2));
    return c;
}
__device__ __forceinline__ C3 to_c3(const Coord& c) {
    return C3{static_cast<std::int32_t>(c.x), static_cast<std::int32_t>(c.y), static_cast<std::int32_t>(c.z)};
}

// Warp-aggregated reservation of n slots on a global counter.  Must be called by
// all 32 lanes of the warp (n may be 0); returns this lane's first slot.
__device__ __forceinline__ unsigned long long warp_reserve(unsigned long long* ctr, unsigned n) {
    const int lane = threadIdx.x & 31;
    unsigned incl = n;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    const unsigned total = __shfl_sync(0xffffffffu, incl, 31);
    unsigned long long base = 0;
    if (lane == 31 && total) base = atomicAdd(ctr, static_cast<unsigned long long>(total));
    base = __shfl_sync(0xffffffffu, base, 31);
    return base + incl - n;
}

// Successors at fixed positions 2*b + (sign > 0) over the three axes b (the odd axis
// of the edge never contributes): ascending position == cofacet order, and all
// accesses use compile-time indices (no local-memory arrays).
struct Succ {
    C3 c[6];
    std::uint32_t valid;  // bit k: position k holds a successor
    std::uint32_t term;   // bit k: that successor is a terminal 2-saddle (quad)
    __device__ __forceinline__ int n() const { return __popc(valid); }
    // the successor at the lowest valid position (valid != 0)
    __device__ __forceinline__ C3 first() const {
        const int k = __ffs(valid) - 1;
        C3 r = c[0];
#pragma unroll
        for (int j = 1; j < 6; ++j)
            if (k == j) r = c[j];
        return r;
    }
    __device__ __forceinline__ bool first_is_term() const { return (term >> (__ffs(valid) - 1)) & 1u; }
    // the successor at position k (runtime k, select chain: no local memory)
    __device__ __forceinline__ C3 at(int k) const {
        C3 r = c[0];
#pragma unroll
        for (int j = 1; j < 6; ++j)
            if (k == j) r = c[j];
        return r;
    }
};

// saddle_graph.cpp:10-24 on coordinates (no id <-> coordinate divisions).
__device__ __forceinline__ Succ successors(const std::uint8_t* __restrict__ codes, const Dims& d,
                                           const C3& e) {
    Succ s;
    s.valid = 0;
    s.term = 0;
    const std::int32_t co[3] = {e.x, e.y, e.z};
    const std::int64_t ext[3] = {d.ex, d.ey, d.ez};
    const std::int64_t eid = cell_id(d, e);
    const std::int64_t step[3] = {1, d.ex, d.exy};
#pragma unroll
    for (int b = 0; b < 3; ++b) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int k = 2 * b + h, sgn = h ? 1 : -1;
            s.c[k] = e;
            if (co[b] & 1) continue;
            if (h == 0 ? co[b] == 0 : co[b] == ext[b] - 1) continue;
            const std::uint8_t code = codes[eid + sgn * step[b]];
            C3 q = e;
            if (b == 0) q.x += sgn;
            else if (b == 1) q.y += sgn;
            else q.z += sgn;
            if (code == kCritical) {
                s.valid |= 1u << k;
                s.term |= 1u << k;
                s.c[k] = q;
            } else if (paired_with_facet(code)) {
                const int dir = code - kFacetBase, ax = dir >> 1, ps = (dir & 1) ? 1 : -1;
                C3 o = q;
                if (ax == 0) o.x += ps;
                else if (ax == 1) o.y += ps;
                else o.z += ps;
                if (o.x != e.x || o.y != e.y || o.z != e.z) {
                    s.valid |= 1u << k;
                    s.c[k] = o;
                }
            }
        }
    }
    return s;
}

template <typename IdT>
__global__ void k_bfs_sources(const std::uint8_t* __restrict__ codes, Dims d,
                              const IdT* __restrict__ src, std::uint64_t n,
                              unsigned int* __restrict__ bitmap, std::uint32_t* __restrict__ frontier,
                              unsigned int* bad) {
    GRID_STRIDE(i, n) {
        const std::uint64_t e = src[i];
        if (e >= d.n_cells) {
            *bad = 1u;
            continue;
        }
        const Coord c = unpack(d, e);
        if (codes[e] != kCritical || cell_dim(c) != 1) {
            *bad = 1u;
            continue;
        }
        const std::uint32_t de = edge_dense(d, to_c3(c));
        atomicOr(&bitmap[de >> 5], 1u << (de & 31));
        frontier[i] = de;
    }
}

// All BFS levels in one cooperative launch.  cnt[0] holds the source count, cnt[1]
// must be 0.  stats[0] = levels, stats[1] = nodes visited.
__global__ void __launch_bounds__(kThreads)
k_bfs_persistent(const std::uint8_t* __restrict__ codes, Dims d, unsigned int* __restrict__ bitmap,
                 std::uint32_t* __restrict__ fa, std::uint32_t* __restrict__ fb,
                 unsigned long long* __restrict__ cnt, unsigned long long* __restrict__ stats) {
    cg::grid_group g = cg::this_grid();
    std::uint32_t* cur = fa;
    std::uint32_t* nxt = fb;
    unsigned long long ncur = *reinterpret_cast<volatile unsigned long long*>(&cnt[0]);
    unsigned long long total = ncur;
    int level = 0;
    const std::uint64_t stride = static_cast<std::uint64_t>(gridDim.x) * blockDim.x;
    while (ncur) {
        unsigned long long* next_cnt = &cnt[(level + 1) % 3];
        if (g.thread_rank() == 0) cnt[(level + 2) % 3] = 0;
        for (std::uint64_t base = (blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x) & ~31ull;
             base < ncur; base += stride) {
            const std::uint64_t j = base + (threadIdx.x & 31);
            std::uint32_t de[6];
            std::uint32_t won = 0;
            if (j < ncur) {
                const Succ s = successors(codes, d, edge_coord(d, cur[j]));
                const std::uint32_t edges = s.valid & ~s.term;
#pragma unroll
                for (int k = 0; k < 6; ++k) {
                    de[k] = edge_dense(d, s.c[k]);
                    if (!((edges >> k) & 1u)) continue;
                    const unsigned bit = 1u << (de[k] & 31);
                    if (bitmap[de[k] >> 5] & bit) continue;  // cheap pre-check
                    if (atomicOr(&bitmap[de[k] >> 5], bit) & bit) continue;
                    won |= 1u << k;
                }
            }
            const unsigned long long at = warp_reserve(next_cnt, __popc(won));
#pragma unroll
            for (int k = 0; k < 6; ++k)
                if ((won >> k) & 1u) nxt[at + __popc(won & ((1u << k) - 1))] = de[k];
        }
        g.sync();
        ncur = *reinterpret_cast<volatile unsigned long long*>(next_cnt);
        total += ncur;
        ++level;
        std::uint32_t* t = cur;
        cur = nxt;
        nxt = t;
    }
    if (g.thread_rank() == 0) {
        stats[0] = static_cast<unsigned long long>(level);
        stats[1] = total;
    }
}

// The API's marked bytes (saddle_graph.hpp:45-50): visited edges, the quads they
// were entered through (their pair partners), and the discovered 2-saddles.
__global__ void k_marked_bytes(const std::uint8_t* __restrict__ codes, Dims d,
                               const unsigned int* __restrict__ bitmap, std::uint64_t nwords,
                               std::uint8_t* __restrict__ marked) {
    GRID_STRIDE(w, nwords) {
        unsigned int bits = bitmap[w];
        while (bits) {
            const int b = __ffs(bits) - 1;
            bits &= bits - 1;
            const std::uint32_t de = static_cast<std::uint32_t>(w * 32 + b);
            const C3 c = edge_coord(d, de);
            const std::int64_t id = cell_id(d, c);
            marked[id] = 1;
            const std::uint8_t k = codes[id];
            if (k != kCritical) marked[partner_of(d, id, k)] = 1;
            const Succ s = successors(codes, d, c);
#pragma unroll
            for (int q = 0; q < 6; ++q)
                if ((s.term >> q) & 1u) marked[cell_id(d, s.c[q])] = 1;
        }
    }
}

// tmap[quad dense(list[k])] = k
template <typename IdT>
__global__ void k_scatter_quad_rank(const IdT* __restrict__ list, std::uint64_t n, Dims d,
                                    std::uint32_t* __restrict__ tmap) {
    GRID_STRIDE(k, n) tmap[quad_dense(d, to_c3(unpack(d, list[k])))] = static_cast<std::uint32_t>(k);
}

// Junctions (saddle_graph.cpp:126-133): visited non-critical edges with > 1
// successor.  Counting pass over the visited bitmap, 32 nodes per thread.
__global__ void k_junction_count(const std::uint8_t* __restrict__ codes, Dims d,
                                 const unsigned int* __restrict__ bitmap, std::uint64_t nwords,
                                 std::uint32_t* __restrict__ per_word) {
    GRID_STRIDE(w, nwords) {
        unsigned int bits = bitmap[w];
        std::uint32_t n = 0;
        while (bits) {
            const int b = __ffs(bits) - 1;
            bits &= bits - 1;
            const C3 c = edge_coord(d, static_cast<std::uint32_t>(w * 32 + b));
            if (codes[cell_id(d, c)] == kCritical) continue;
            n += successors(codes, d, c).n() > 1;
        }
        per_word[w] = n;
    }
}

__global__ void k_junction_write(const std::uint8_t* __restrict__ codes, Dims d,
                                 const unsigned int* __restrict__ bitmap, std::uint64_t nwords,
                                 const std::uint64_t* __restrict__ off, std::uint32_t* __restrict__ jlist,
                                 std::uint32_t* __restrict__ jidx) {
    GRID_STRIDE(w, nwords) {
        unsigned int bits = bitmap[w];
        std::uint64_t at = off[w];
        while (bits) {
            const int b = __ffs(bits) - 1;
            bits &= bits - 1;
            const std::uint32_t de = static_cast<std::uint32_t>(w * 32 + b);
            const C3 c = edge_coord(d, de);
            if (codes[cell_id(d, c)] == kCritical) continue;
            if (successors(codes, d, c).n() > 1) {
                jlist[at] = de;
                jidx[de] = static_cast<std::uint32_t>(at);
                ++at;
            }
        }
    }
}

// Per origin (junctions: list of dense edges; sources: id list), the <= 4 branch
// destinations: every branch is walked to its end (saddle_graph.cpp:139-202):
// terminal 2-saddle -> kTerm|rank, junction -> junction index, dead end -> kNone.
// Junction origins also count pending junction branches and predecessor
// in-degrees for Kahn.
template <typename IdT>
__global__ void k_origin_dests(const std::uint8_t* __restrict__ codes, Dims d,
                               const std::uint32_t* __restrict__ jlist, const IdT* __restrict__ srcs,
                               std::uint64_t n, const std::uint32_t* __restrict__ jidx,
                               const std::uint32_t* __restrict__ tmap, std::uint32_t* __restrict__ dest,
                               std::uint32_t* __restrict__ pending, std::uint32_t* __restrict__ indeg,
                               unsigned int* __restrict__ flags) {
    GRID_STRIDE(i, n) {
        const C3 o = jlist ? edge_coord(d, jlist[i]) : to_c3(unpack(d, srcs[i]));
        const Succ s = successors(codes, d, o);
        std::uint32_t dd[4] = {kNone, kNone, kNone, kNone};
        std::uint32_t pend = 0;
        int nd = 0;
#pragma unroll 1
        for (std::uint32_t todo = s.valid; todo; todo &= todo - 1) {
            const int b = __ffs(todo) - 1;
            const C3 sb = s.at(b);
            std::uint32_t t;
            if ((s.term >> b) & 1u) {
                t = kTerm | tmap[quad_dense(d, sb)];
            } else {
                // the walk stops AT a junction, else follows the junction-free chain
                C3 cur = sb;
                t = kNone;
                for (std::uint64_t steps = 0;; ++steps) {
                    const Succ nx = successors(codes, d, cur);
                    const int nn = nx.n();
                    if (nn > 1) {
                        t = jidx[edge_dense(d, cur)];
                        break;
                    }
                    if (nn == 0) break;
                    if (nx.first_is_term()) {
                        t = kTerm | tmap[quad_dense(d, nx.first())];
                        break;
                    }
                    cur = nx.first();
                    if (steps > d.n_cells) {
                        flags[2] = 1u;  // cycle: invalid gradient (saddle_graph.cpp:173-174)
                        break;
                    }
                }
            }
            // append in branch order (constant-index selects, no local memory)
            dd[0] = nd == 0 ? t : dd[0];
            dd[1] = nd == 1 ? t : dd[1];
            dd[2] = nd == 2 ? t : dd[2];
            dd[3] = nd == 3 ? t : dd[3];
            ++nd;
            if (!(t & kTerm)) {
                ++pend;
                if (indeg) atomicAdd(&indeg[t], 1u);
            }
        }
        reinterpret_cast<uint4*>(dest)[i] = make_uint4(dd[0], dd[1], dd[2], dd[3]);
        if (pending) pending[i] = pend;
    }
}

__global__ void k_fill_rev(const std::uint32_t* __restrict__ dest, std::uint64_t nj,
                           const std::uint64_t* __restrict__ roff, std::uint32_t* __restrict__ cursor,
                           std::uint32_t* __restrict__ rsrc) {
    GRID_STRIDE(i, nj) {
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const std::uint32_t t = dest[4 * i + b];
            if (t & kTerm) continue;
            const std::uint32_t at = atomicAdd(&cursor[t], 1u);
            rsrc[roff[t] + at] = static_cast<std::uint32_t>(i);
        }
    }
}

__global__ void k_initial_frontier(const std::uint32_t* __restrict__ pending, std::uint64_t nj,
                                   std::uint32_t* __restrict__ frontier,
                                   unsigned long long* __restrict__ count) {
    const std::uint64_t stride = static_cast<std::uint64_t>(gridDim.x) * blockDim.x;
    for (std::uint64_t base = (blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x) & ~31ull;
         base < nj; base += stride) {
        const std::uint64_t i = base + (threadIdx.x & 31);
        const bool ready = i < nj && pending[i] == 0;
        const unsigned long long at = warp_reserve(count, ready ? 1u : 0u);
        if (ready) frontier[at] = static_cast<std::uint32_t>(i);
    }
}

struct Pool {
    std::uint32_t* key;
    std::uint64_t* cnt;
    unsigned long long* top;
    std::uint64_t cap;
};

__device__ __forceinline__ bool add_ovf(std::uint64_t a, std::uint64_t b, std::uint64_t* r) {
    *r = a + b;
    return *r < a;
}
__device__ __forceinline__ bool mul_ovf(std::uint64_t a, std::uint64_t b, std::uint64_t* r) {
    *r = a * b;
    return __umul64hi(a, b) != 0;
}

// K-way merge of up to 4 sorted (key, count) lists scaled by mult.  A terminal
// branch is a one-element list.  With okey == nullptr only the length is counted.
struct MergeIn {  // slot b = branch b of the origin (empty when len[b] == 0)
    const std::uint32_t* key[4];
    const std::uint64_t* cnt[4];
    std::uint32_t len[4];
    std::uint32_t one_key[4];
    std::uint64_t mult[4];
};

__device__ __forceinline__ std::uint32_t kway_merge(const MergeIn& in, std::uint32_t* okey,
                                                    std::uint64_t* ocnt, unsigned int* ovf) {
    std::uint32_t pos[4] = {0, 0, 0, 0};
    std::uint32_t out = 0;
    for (;;) {
        std::uint32_t best = 0xffffffffu;
        bool any = false;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            if (pos[b] >= in.len[b]) continue;
            const std::uint32_t kk = in.key[b] ? in.key[b][pos[b]] : in.one_key[b];
            if (!any || kk < best) best = kk;
            any = true;
        }
        if (!any) break;
        std::uint64_t sum = 0;
        bool o = false;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            if (pos[b] >= in.len[b]) continue;
            const std::uint32_t kk = in.key[b] ? in.key[b][pos[b]] : in.one_key[b];
            if (kk != best) continue;
            const std::uint64_t c = in.cnt[b] ? in.cnt[b][pos[b]] : 1ull;
            std::uint64_t pr;
            o |= mul_ovf(c, in.mult[b], &pr);
            o |= add_ovf(sum, pr, &sum);
            ++pos[b];
        }
        if (o) *ovf = 1u;
        if (okey) {
            okey[out] = best;
            ocnt[out] = sum;
        }
        ++out;
    }
    return out;
}

__device__ __forceinline__ void gather_inputs(const std::uint32_t* __restrict__ dest, std::uint64_t i,
                                              const std::uint64_t* __restrict__ poff,
                                              const std::uint32_t* __restrict__ plen, const Pool& pool,
                                              MergeIn& in) {
    const uint4 d4 = reinterpret_cast<const uint4*>(dest)[i];
    const std::uint32_t dd[4] = {d4.x, d4.y, d4.z, d4.w};
#pragma unroll
    for (int b = 0; b < 4; ++b) {
        const std::uint32_t t = dd[b];
        in.mult[b] = 1;
        in.one_key[b] = t & ~kTerm;
        in.key[b] = nullptr;
        in.cnt[b] = nullptr;
        in.len[b] = 0;
        if (t == kNone) continue;
        if (t & kTerm) {
            in.len[b] = 1;
        } else {
            in.key[b] = pool.key + poff[t];
            in.cnt[b] = pool.cnt + poff[t];
            in.len[b] = plen[t];
        }
    }
}

// All Kahn levels in one cooperative launch.  cnt[0] = initial frontier size,
// cnt[1] = 0.  stats[0] = levels, stats[1] = junctions processed.  flags[0]:
// overflow, flags[1]: pool exhausted (the host grows the pool and reruns).
__global__ void __launch_bounds__(kThreads)
k_kahn_persistent(const std::uint32_t* __restrict__ dest, std::uint64_t* __restrict__ poff,
                  std::uint32_t* __restrict__ plen, Pool pool, const std::uint64_t* __restrict__ roff,
                  const std::uint32_t* __restrict__ rcnt, const std::uint32_t* __restrict__ rsrc,
                  std::uint32_t* __restrict__ pending, std::uint32_t* __restrict__ fa,
                  std::uint32_t* __restrict__ fb, unsigned long long* __restrict__ cnt,
                  unsigned int* __restrict__ flags, unsigned long long* __restrict__ stats) {
    cg::grid_group g = cg::this_grid();
    std::uint32_t* cur = fa;
    std::uint32_t* nxt = fb;
    unsigned long long ncur = *reinterpret_cast<volatile unsigned long long*>(&cnt[0]);
    unsigned long long done = 0;
    int level = 0;
    const std::uint64_t stride = static_cast<std::uint64_t>(gridDim.x) * blockDim.x;
    while (ncur) {
        unsigned long long* next_cnt = &cnt[(level + 1) % 3];
        if (g.thread_rank() == 0) cnt[(level + 2) % 3] = 0;
        for (std::uint64_t base = (blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x) & ~31ull;
             base < ncur; base += stride) {
            const std::uint64_t f = base + (threadIdx.x & 31);
            const bool valid = f < ncur;
            std::uint32_t j = 0, len = 0;
            MergeIn in;
#pragma unroll
            for (int b = 0; b < 4; ++b) in.len[b] = 0;
            if (valid) {
                j = cur[f];
                gather_inputs(dest, j, poff, plen, pool, in);
                len = kway_merge(in, nullptr, nullptr, &flags[0]);
            }
            const unsigned long long at = warp_reserve(pool.top, len);
            if (valid) {
                if (at + len > pool.cap) {
                    flags[1] = 1u;
                    poff[j] = 0;
                    plen[j] = 0;
                } else {
                    kway_merge(in, pool.key + at, pool.cnt + at, &flags[0]);
                    poff[j] = at;
                    plen[j] = len;
                }
            }
            std::uint64_t r0 = 0;
            std::uint32_t rn = 0;
            if (valid) {
                r0 = roff[j];
                rn = rcnt[j];
            }
            for (;;) {
                std::uint32_t rel[4];
                unsigned nrel = 0;
                while (rn && nrel < 4) {
                    const std::uint32_t p = rsrc[r0++];
                    --rn;
                    if (atomicSub(&pending[p], 1u) == 1u) rel[nrel++] = p;
                }
                const unsigned long long q = warp_reserve(next_cnt, nrel);
                for (unsigned k = 0; k < nrel; ++k) nxt[q + k] = rel[k];
                if (!__any_sync(0xffffffffu, rn != 0)) break;
            }
        }
        g.sync();
        done += ncur;
        ncur = *reinterpret_cast<volatile unsigned long long*>(next_cnt);
        ++level;
        std::uint32_t* t = cur;
        cur = nxt;
        nxt = t;
    }
    if (g.thread_rank() == 0) {
        stats[0] = static_cast<unsigned long long>(level);
        stats[1] = done;
    }
}

// Sources: pass 1 lengths, pass 2 writes (one_saddle rank, two_saddle rank, paths).
__global__ void k_source_len(const std::uint32_t* __restrict__ dest, std::uint64_t n1,
                             const std::uint64_t* __restrict__ poff, const std::uint32_t* __restrict__ plen,
                             Pool pool, std::uint32_t* __restrict__ len, unsigned int* __restrict__ flags) {
    GRID_STRIDE(i, n1) {
        MergeIn in;
        gather_inputs(dest, i, poff, plen, pool, in);
        len[i] = kway_merge(in, nullptr, nullptr, &flags[0]);
    }
}

__global__ void k_source_write(const std::uint32_t* __restrict__ dest, std::uint64_t n1,
                               const std::uint64_t* __restrict__ poff, const std::uint32_t* __restrict__ plen,
                               Pool pool, const std::uint64_t* __restrict__ off,
                               std::uint32_t* __restrict__ o_one, std::uint32_t* __restrict__ o_two,
                               std::uint64_t* __restrict__ o_cnt, unsigned int* __restrict__ flags) {
    GRID_STRIDE(i, n1) {
        MergeIn in;
        gather_inputs(dest, i, poff, plen, pool, in);
        const std::uint64_t at = off[i];
        const std::uint32_t len = kway_merge(in, o_two + at, o_cnt + at, &flags[0]);
        for (std::uint32_t k = 0; k < len; ++k) o_one[at + k] = static_cast<std::uint32_t>(i);
    }
}

int coop_grid(const void* fn, int num_sms, int* grid) {
    int per_sm = 0;
    MSC3D_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kThreads, 0));
    if (per_sm <= 0) return MSC3D_ERR_CUDA;
    *grid = per_sm * num_sms;
    return MSC3D_OK;
}

}  // namespace

// ---------------------------------------------------------------------------------
// host wrappers
// ---------------------------------------------------------------------------------

int launch_bfs_sources(const std::uint8_t* codes, const Dims& d, const void* src, std::uint64_t n,
                       int id_width, unsigned int* bitmap, std::uint32_t* frontier, unsigned int* bad,
                       cudaStream_t s, int num_sms) {
    if (n == 0) return MSC3D_OK;
    if (id_width == 4)
        k_bfs_sources<std::uint32_t><<<grid_for(n, num_sms), kThreads, 0, s>>>(
            codes, d, static_cast<const std::uint32_t*>(src), n, bitmap, frontier, bad);
    else
        k_bfs_sources<std::uint64_t><<<grid_for(n, num_sms), kThreads, 0, s>>>(
            codes, d, static_cast<const std::uint64_t*>(src), n, bitmap, frontier, bad);
    count_launch();
    MSC3D_CUDA_TRY(cudaGetLastError());
    return MSC3D_OK;
}

int launch_bfs_persistent(const std::uint8_t* codes, const Dims& d, unsigned int* bitmap,
                          std::uint32_t* fa, std::uint32_t* fb, unsigned long long* cnt,
                          unsigned long long* stats, cudaStream_t s, int num_sms) {
    int grid = 0;
    const int rc = coop_grid(reinterpret_cast<const void*>(k_bfs_persistent), num_sms, &grid);
    if (rc != MSC3D_OK) return rc;
    Dims dd = d;
    const std::uint8_t* c = codes;
    void* args[] = {&c, &dd, &bitmap, &fa, &fb, &cnt, &stats};
    MSC3D_CUDA_TRY(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k_bfs_persistent),
                                               dim3(grid), dim3(kThreads), args, 0, s));
    count_launch();
    return MSC3D_OK;
}

int launch_marked_bytes(const std::uint8_t* codes, const Dims& d, const unsigned int* bitmap,
                        std::uint64_t nwords, std::uint8_t* marked, cudaStream_t s, int num_sms) {
    if (nwords == 0) return MSC3D_OK;
    k_marked_bytes<<<grid_for(nwords, num_sms), kThreads, 0, s>>>(codes, d, bitmap, nwords, marked);
    count_launch();
    MSC3D_CUDA_TRY(cudaGetLastError());
    return MSC3D_OK;
}

int launch_scatter_quad_rank(const void* list, std::uint64_t n, int id_width, const Dims& d,
                             std::uint32_t* tmap, cudaStream_t s, int num_sms) {
    if (n == 0) return MSC3D_OK;
    if (id_width == 4)
        k_scatter_quad_rank<std::uint32_t><<<grid_for(n, num_sms), kThreads, 0, s>>>(
            static_cast<const std::uint32_t*>(list), n, d, tmap);
    else
        k_scatter_quad_rank<std::uint64_t><<<grid_for(n, num_sms), kThreads, 0, s>>>(
            static_cast<const std::uint64_t*>(list), n, d, tmap);
    count_launch();
    MSC3D_CUDA_TRY(cudaGetLastError());
    return MSC3D_OK;
}

int launch_junction_count(const std::uint8_t* codes, const Dims& d, const unsigned int* bitmap,
                          std::uint64_t nwords, std::uint32_t* per_word, cudaStream_t s, int num_sms) {
    if (nwords == 0) return MSC3D_OK;
    k_junction_count<<<grid_for(nwords, num_sms, 32), kThreads, 0, s>>>(codes, d, bitmap, nwords, per_word);
    count_launch();
    MSC3D_CUDA_TRY(cudaGetLastError());
    return MSC3D_OK;
}

int launch_junction_write(const std::uint8_t* codes, const Dims& d, const unsigned int* bitmap,
                          std::uint64_t nwords, const std::uint64_t* off, std::uint32_t* jlist,
                          std::uint32_t* jidx, cudaStream_t s, int num_sms) {
    if (nwords == 0) return MSC3D_OK;
    k_junction_write<<<grid_for(nwords, num_sms, 32), kThreads, 0, s>>>(codes, d, bitmap, nwords, off,
                                                                        jlist, jidx);
    count_launch();
    MSC3D_CUDA_TRY(cudaGetLastError());
    return MSC3D_OK;
}

int launch_origin_dests(const std::uint8_t* codes, const Dims& d, const std::uint32_t* jlist,
                        const void* srcs, int id_width, std::uint64_t n, const std::uint32_t* jidx,
                        const std::uint32_t* tmap, std::uint32_t* dest, std::uint32_t* pending,
                        std::uint32_t* indeg, unsigned int* flags, cudaStream_t s, int num_sms) {
    if (n == 0) return MSC3D_OK;
    if (id_width == 4)
        k_origin_dests<std::uint32_t><<<grid_for(n, num_sms, 32), kThreads, 0, s>>>(
            codes, d, jlist, static_cast<const std::uint32_t*>(srcs), n, jidx, tmap, dest, pending,
            indeg, flags);
    else
        k_origin_dests<std::uint64_t><<<grid_for(n, num_sms, 32), kThreads, 0, s>>>(
            codes, d, jlist, static_cast<const std::uint64_t*>(srcs), n, jidx, tmap, dest, pending,
            indeg, flags);
    count_launch();
    MSC3D_CUDA_TRY(cudaGetLastError());
    return MSC3D_OK;
}

int launch_fill_rev(const std::uint32_t* dest, std::uint64_t nj, const std::uint64_t* roff,
                    std::uint32_t* cursor, std::uint32_t* rsrc, cudaStream_t s, int num_sms) {
    if (nj == 0) return MSC3D_OK;
    k_fill_rev<<<grid_for(nj, num_sms), kThreads, 0, s>>>(dest, nj, roff, cursor, rsrc);
    count_launch();
    MSC3D_CUDA_TRY(cudaGetLastError());
    return MSC3D_OK;
}

int launch_initial_frontier(const std::uint32_t* pending, std::uint64_t nj, std::uint32_t* frontier,
                            unsigned long long* count, cudaStream_t s, int num_sms) {
    if (nj == 0) return MSC3D_OK;
    k_initial_frontier<<<grid_for(nj, num_sms), kThreads, 0, s>>>(pending, nj, frontier, count);
    count_launch();
    MSC3D_CUDA_TRY(cudaGetLastError());
    return MSC3D_OK;
}

int launch_kahn_persistent(const std::uint32_t* dest, std::uint64_t* poff, std::uint32_t* plen,
                           std::uint32_t* pkey, std::uint64_t* pcnt, unsigned long long* ptop,
                           std::uint64_t pcap, const std::uint64_t* roff, const std::uint32_t* rcnt,
                           const std::uint32_t* rsrc, std::uint32_t* pending, std::uint32_t* fa,
                           std::uint32_t* fb, unsigned long long* cnt, unsigned int* flags,
                           unsigned long long* stats, cudaStream_t s, int num_sms) {
    int grid = 0;
    const int rc = coop_grid(reinterpret_cast<const void*>(k_kahn_persistent), num_sms, &grid);
    if (rc != MSC3D_OK) return rc;
    Pool pool{pkey, pcnt, ptop, pcap};
    void* args[] = {&dest, &poff, &plen, &pool, &roff, &rcnt, &rsrc, &pending, &fa, &fb, &cnt, &flags, &stats};
    MSC3D_CUDA_TRY(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k_kahn_persistent),
                                               dim3(grid), dim3(kThreads), args, 0, s));
    count_launch();
    return MSC3D_OK;
}

int launch_source_len(const std::uint32_t* dest, std::uint64_t n1, const std::uint64_t* poff,
                      const std::uint32_t* plen, const std::uint32_t* pkey, const std::uint64_t* pcnt,
                      std::uint32_t* len, unsigned int* flags, cudaStream_t s, int num_sms) {
    if (n1 == 0) return MSC3D_OK;
    Pool pool{const_cast<std::uint32_t*>(pkey), const_cast<std::uint64_t*>(pcnt), nullptr, 0};
    k_source_len<<<grid_for(n1, num_sms), kThreads, 0, s>>>(dest, n1, poff, plen, pool, len, flags);
    count_launch();
    MSC3D_CUDA_TRY(cudaGetLastError());
    return MSC3D_OK;
}

int launch_source_write(const std::uint32_t* dest, std::uint64_t n1, const std::uint64_t* poff,
                        const std::uint32_t* plen, const std::uint32_t* pkey,
                        const std::uint64_t* pcnt, const std::uint64_t* off, std::uint32_t* o_one,
                        std::uint32_t* o_two, std::uint64_t* o_cnt, unsigned int* flags,
                        cudaStream_t s, int num_sms) {
    if (n1 == 0) return MSC3D_OK;
    Pool pool{const_cast<std::uint32_t*>(pkey), const_cast<std::uint64_t*>(pcnt), nullptr, 0};
    k_source_write<<<grid_for(n1, num_sms), kThreads, 0, s>>>(dest, n1, poff, plen, pool, off,
                                                             o_one, o_two, o_cnt, flags);
    count_launch();
    MSC3D_CUDA_TRY(cudaGetLastError());
    return MSC3D_OK;
}

}  // namespace msc3d_dev

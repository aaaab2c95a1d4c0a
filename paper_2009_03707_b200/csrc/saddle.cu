// Saddle-graph helpers shared by the pipeline (stages.cu) and the stage-level
// build_minor (minor.cu), after proj/src/saddle_graph.cpp:
//   * k_bfs_sources    -- validate the BFS sources (critical 1-cells,
//                         saddle_graph.cpp:29-41), set their visited bits, seed the frontier;
//   * k_marked_bytes   -- MarkedSubgraph::marked bytes from the visited bitmap (edges,
//                         the quads they were entered through, discovered 2-saddles);
//   * k_scatter_quad_rank -- 2-saddle quad -> rank in its sorted list;
//   * k_origin_dests   -- per 1-saddle / junction branch, the walk to its end
//                         (2-saddle, junction or dead end), saddle_graph.cpp:139-202.
// Node space: DAG nodes are 1-cells indexed by the dense edge id de = 3 * (lower
// vertex) + axis.  Successors (saddle_graph.cpp:10-24) are recomputed from the pair
// codes here; the pipeline's own BFS / walks / counting (dag.cu) use 2-byte
// successor words instead.
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

}  // namespace msc3d_dev

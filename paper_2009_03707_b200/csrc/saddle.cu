// Saddle-saddle stages: DAG successors, reachability, chain contraction, minor
// edges, and 2-saddle-keyed path counting (proj/src/saddle_graph.cpp,
// proj/src/path_matrix.cpp), re-designed for the device.
//
// Node store.  Every 1-cell reached from a 1-saddle becomes a node, numbered in
// discovery order (sources first).  Nodes are kept as u32 "dense edge" indices
// (3 * lower-vertex + axis), and nid[dense edge] maps back to the node number; it
// is written only when a node is claimed and read only for claimed nodes, so it
// is never initialised.
//
// Successors (saddle_graph.cpp:10-24): for each cofacet quad q of e in cofacet
// order, q critical -> terminal 2-saddle q; q paired with a facet edge e' != e ->
// edge e'; q paired with a cube -> nothing.
//
// Reachability (saddle_graph.cpp:26-86): level-synchronous frontier expansion;
// a node is claimed with an atomic OR on its marked byte (so the marked SET is the
// reference's, whatever the schedule), and the quad it was entered through is
// marked with it.
//
// Counting.  The reference contracts junction-free paths into a minor and runs
// sparse matrix products A* = A(I + B + B^2 ...), A*B* + D.  Here: (1) chain
// contraction by pointer jumping over out-degree-1 nodes (the same forest trick as
// the extrema), (2) per junction, the sparse vector P(j) of path counts to
// 2-saddles, computed in reverse topological order (Kahn's algorithm on the
// junction graph, one frontier per level) by merging the successors' vectors, and
// (3) per 1-saddle the same merge written straight to the output.  Total work is
// the sum of backward cone sizes of the 2-saddles (measured 1.3-1.9x the node count
// on the BASELINE fields, SURVEY/BASELINE config data).  Counts are exact u64 with
// sticky overflow detection.
#include "common.cuh"
#include "kernels.cuh"

namespace msc3d_dev {

namespace {

constexpr int kThreads = 256;
constexpr std::uint32_t kTerm = 0x80000000u;
constexpr std::uint32_t kNone = 0xffffffffu;

inline unsigned grid_for(std::uint64_t n, int num_sms, int per_sm = 16) {
    const std::uint64_t need = (n + kThreads - 1) / kThreads;
    return static_cast<unsigned>(std::max<std::uint64_t>(
        1, std::min<std::uint64_t>(need, static_cast<std::uint64_t>(num_sms) * per_sm)));
}

#define GRID_STRIDE(i, n)                                                                       \
    for (std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x; \
         i < (n); i += static_cast<std::uint64_t>(gridDim.x) * blockDim.x)

__device__ __forceinline__ std::uint32_t edge_dense(const Dims& d, const Coord& c) {
    const int axis = (c.x & 1) ? 0 : ((c.y & 1) ? 1 : 2);
    return 3u * static_cast<std::uint32_t>((c.x >> 1) + d.nx * ((c.y >> 1) + d.ny * (c.z >> 1))) + axis;
}
__device__ __forceinline__ std::uint32_t quad_dense(const Dims& d, const Coord& c) {
    const int axis = !(c.x & 1) ? 0 : (!(c.y & 1) ? 1 : 2);
    return 3u * static_cast<std::uint32_t>((c.x >> 1) + d.nx * ((c.y >> 1) + d.ny * (c.z >> 1))) + axis;
}
__device__ __forceinline__ Coord edge_coord(const Dims& d, std::uint32_t de) {
    const std::uint32_t v = de / 3, a = de - 3 * v;
    const std::uint64_t vx = v % d.nx, r = v / d.nx, vy = r % d.ny, vz = r / d.ny;
    Coord c;
    c.x = 2 * vx + (a == 0);
    c.y = 2 * vy + (a == 1);
    c.z = 2 * vz + (a == 2);
    return c;
}

// Byte-granular atomic OR on a u8 array; returns the previous byte.
__device__ __forceinline__ std::uint8_t atomic_or_byte(std::uint8_t* base, std::uint64_t i,
                                                       std::uint8_t v) {
    auto* w = reinterpret_cast<unsigned int*>(base + (i & ~3ull));
    const int sh = 8 * static_cast<int>(i & 3);
    const unsigned int old = atomicOr(w, static_cast<unsigned int>(v) << sh);
    return static_cast<std::uint8_t>(old >> sh);
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

// Successor enumeration of edge cell e (coords c): calls f(is_terminal, cell id).
template <typename F>
__device__ __forceinline__ void for_successors(const std::uint8_t* __restrict__ codes, const Dims& d,
                                               const Coord& c, F&& f) {
    const std::int64_t e = static_cast<std::int64_t>(pack(d, c.x, c.y, c.z));
    const std::int64_t co[3] = {c.x, c.y, c.z};
    const std::int64_t ext[3] = {d.ex, d.ey, d.ez};
    const std::int64_t step[3] = {1, d.ex, d.exy};
#pragma unroll
    for (int b = 0; b < 3; ++b) {
        if (co[b] & 1) continue;
#pragma unroll
        for (int sgn = -1; sgn <= 1; sgn += 2) {
            if (sgn < 0 ? co[b] == 0 : co[b] == ext[b] - 1) continue;
            const std::int64_t q = e + sgn * step[b];
            const std::uint8_t k = codes[q];
            if (k == kCritical) {
                f(true, q);
            } else if (paired_with_facet(k)) {
                const std::int64_t o = partner_of(d, q, k);
                if (o != e) f(false, o);
            }
        }
    }
}

template <typename IdT>
__global__ void k_mark_sources(const std::uint8_t* __restrict__ codes, Dims d,
                               const IdT* __restrict__ src, std::uint64_t n,
                               std::uint8_t* __restrict__ marked, std::uint32_t* __restrict__ nodes,
                               std::uint32_t* __restrict__ nid, unsigned int* bad) {
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
        atomic_or_byte(marked, e, 1);
        const std::uint32_t de = edge_dense(d, c);
        nodes[i] = de;
        nid[de] = static_cast<std::uint32_t>(i);
    }
}

__global__ void k_bfs_level(const std::uint8_t* __restrict__ codes, Dims d,
                            std::uint8_t* __restrict__ marked, std::uint32_t* __restrict__ nodes,
                            std::uint64_t begin, std::uint64_t end,
                            unsigned long long* __restrict__ tail, std::uint32_t* __restrict__ nid) {
    const std::uint64_t n = end - begin;
    const std::uint64_t stride = static_cast<std::uint64_t>(gridDim.x) * blockDim.x;
    for (std::uint64_t base = (blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x) & ~31ull;
         base < n; base += stride) {
        const std::uint64_t j = base + (threadIdx.x & 31);
        std::uint32_t won[4];
        unsigned nwon = 0;
        if (j < n) {
            const Coord c = edge_coord(d, nodes[begin + j]);
            for_successors(codes, d, c, [&](bool term, std::int64_t x) {
                if (atomic_or_byte(marked, static_cast<std::uint64_t>(x), 1) || term) return;
                // claimed: mark the quad we came through (its pair partner)
                const std::uint8_t kx = codes[x];
                atomic_or_byte(marked, static_cast<std::uint64_t>(partner_of(d, x, kx)), 1);
                won[nwon++] = edge_dense(d, unpack(d, static_cast<std::uint64_t>(x)));
            });
        }
        const unsigned long long at = warp_reserve(tail, nwon);
        for (unsigned k = 0; k < nwon; ++k) {
            nodes[at + k] = won[k];
            nid[won[k]] = static_cast<std::uint32_t>(at + k);
        }
    }
}

// tmap[quad dense(list[k])] = k
template <typename IdT>
__global__ void k_scatter_quad_rank(const IdT* __restrict__ list, std::uint64_t n, Dims d,
                                    std::uint32_t* __restrict__ tmap) {
    GRID_STRIDE(k, n) tmap[quad_dense(d, unpack(d, list[k]))] = static_cast<std::uint32_t>(k);
}

// Successor table of every node: 4 slots (kNone-padded), terminals as kTerm|rank.
__global__ void k_node_succ(const std::uint8_t* __restrict__ codes, Dims d,
                            const std::uint32_t* __restrict__ nodes, std::uint64_t m,
                            const std::uint32_t* __restrict__ nid,
                            const std::uint32_t* __restrict__ tmap,
                            std::uint32_t* __restrict__ succ, std::uint8_t* __restrict__ outdeg) {
    GRID_STRIDE(k, m) {
        const Coord c = edge_coord(d, nodes[k]);
        std::uint32_t s[4] = {kNone, kNone, kNone, kNone};
        int n = 0;
        for_successors(codes, d, c, [&](bool term, std::int64_t x) {
            const Coord cx = unpack(d, static_cast<std::uint64_t>(x));
            s[n++] = term ? (kTerm | tmap[quad_dense(d, cx)]) : nid[edge_dense(d, cx)];
        });
        reinterpret_cast<uint4*>(succ)[k] = make_uint4(s[0], s[1], s[2], s[3]);
        outdeg[k] = static_cast<std::uint8_t>(n);
    }
}

// Chain pointer: a non-source, non-junction node whose single successor is a
// non-junction edge node continues into it; everything else is a stop.
__global__ void k_chain_ptr(const std::uint32_t* __restrict__ succ, const std::uint8_t* __restrict__ outdeg,
                            std::uint64_t m, std::uint64_t n_src, std::uint32_t* __restrict__ ptr) {
    GRID_STRIDE(k, m) {
        std::uint32_t p = static_cast<std::uint32_t>(k);
        if (k >= n_src && outdeg[k] == 1) {
            const std::uint32_t s = succ[4 * k];
            if (!(s & kTerm) && outdeg[s] <= 1) p = s;
        }
        ptr[k] = p;
    }
}

// Junction flags -> counts for compaction (node order).
__global__ void k_junction_flags(const std::uint8_t* __restrict__ outdeg, std::uint64_t m,
                                 std::uint64_t n_src, std::uint32_t* __restrict__ flag) {
    GRID_STRIDE(k, m) flag[k] = (k >= n_src && outdeg[k] > 1) ? 1u : 0u;
}

__global__ void k_junction_write(const std::uint32_t* __restrict__ flag, const std::uint64_t* __restrict__ off,
                                 std::uint64_t m, std::uint32_t* __restrict__ jlist,
                                 std::uint32_t* __restrict__ jidx) {
    GRID_STRIDE(k, m) {
        if (flag[k]) {
            jlist[off[k]] = static_cast<std::uint32_t>(k);
            jidx[k] = static_cast<std::uint32_t>(off[k]);
        }
    }
}

// Destination of one successor slot: terminal rank, junction index, or none.
__device__ __forceinline__ std::uint32_t branch_dest(std::uint32_t s, const std::uint32_t* __restrict__ succ,
                                                     const std::uint8_t* __restrict__ outdeg,
                                                     const std::uint32_t* __restrict__ stop,
                                                     const std::uint32_t* __restrict__ jidx) {
    if (s == kNone) return kNone;
    if (s & kTerm) return s;
    if (outdeg[s] > 1) return jidx[s];
    const std::uint32_t y = stop[s];
    if (outdeg[y] == 0) return kNone;
    const std::uint32_t s2 = succ[4ull * y];
    if (s2 & kTerm) return s2;
    return jidx[s2];
}

// Per origin (junction list entries, or sources when jlist == nullptr) the 4
// branch destinations.
__global__ void k_origin_dests(const std::uint32_t* __restrict__ jlist, std::uint64_t n,
                               const std::uint32_t* __restrict__ succ, const std::uint8_t* __restrict__ outdeg,
                               const std::uint32_t* __restrict__ stop, const std::uint32_t* __restrict__ jidx,
                               std::uint32_t* __restrict__ dest, std::uint32_t* __restrict__ pending,
                               std::uint32_t* __restrict__ indeg) {
    GRID_STRIDE(i, n) {
        const std::uint64_t k = jlist ? jlist[i] : i;
        const uint4 s4 = reinterpret_cast<const uint4*>(succ)[k];
        const std::uint32_t s[4] = {s4.x, s4.y, s4.z, s4.w};
        std::uint32_t dd[4];
        std::uint32_t pend = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            dd[b] = branch_dest(s[b], succ, outdeg, stop, jidx);
            if (!(dd[b] & kTerm)) {
                ++pend;
                if (indeg) atomicAdd(&indeg[dd[b]], 1u);
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
    GRID_STRIDE(i, nj) {
        if (pending[i] == 0) frontier[atomicAdd(count, 1ull)] = static_cast<std::uint32_t>(i);
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
// branch is a one-element list.  With out == nullptr only the length is counted.
struct MergeIn {
    const std::uint32_t* key[4];
    const std::uint64_t* cnt[4];
    std::uint32_t len[4];
    std::uint32_t one_key[4];
    std::uint64_t mult[4];
    int n;
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
            if (b >= in.n || pos[b] >= in.len[b]) continue;
            const std::uint32_t kk = in.key[b] ? in.key[b][pos[b]] : in.one_key[b];
            if (!any || kk < best) best = kk;
            any = true;
        }
        if (!any) break;
        std::uint64_t sum = 0;
        bool o = false;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            if (b >= in.n || pos[b] >= in.len[b]) continue;
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
    in.n = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
        const std::uint32_t t = dest[4 * i + b];
        if (t == kNone) continue;
        const int k = in.n++;
        in.mult[k] = 1;
        if (t & kTerm) {
            in.key[k] = nullptr;
            in.cnt[k] = nullptr;
            in.len[k] = 1;
            in.one_key[k] = t & ~kTerm;
        } else {
            in.key[k] = pool.key + poff[t];
            in.cnt[k] = pool.cnt + poff[t];
            in.len[k] = plen[t];
            in.one_key[k] = 0;
        }
    }
}

__global__ void k_kahn_level(const std::uint32_t* __restrict__ frontier, std::uint64_t nf,
                             const std::uint32_t* __restrict__ dest, std::uint64_t* __restrict__ poff,
                             std::uint32_t* __restrict__ plen, Pool pool,
                             const std::uint64_t* __restrict__ roff, const std::uint32_t* __restrict__ rcnt,
                             const std::uint32_t* __restrict__ rsrc, std::uint32_t* __restrict__ pending,
                             std::uint32_t* __restrict__ next, unsigned long long* __restrict__ next_count,
                             unsigned int* __restrict__ flags) {
    const std::uint64_t stride = static_cast<std::uint64_t>(gridDim.x) * blockDim.x;
    for (std::uint64_t base = (blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x) & ~31ull;
         base < nf; base += stride) {
        const std::uint64_t f = base + (threadIdx.x & 31);
        const bool valid = f < nf;
        std::uint32_t j = 0, len = 0;
        MergeIn in;
        in.n = 0;
        if (valid) {
            j = frontier[f];
            gather_inputs(dest, j, poff, plen, pool, in);
            len = kway_merge(in, nullptr, nullptr, &flags[0]);
        }
        const unsigned long long at = warp_reserve(pool.top, len);
        if (valid) {
            if (at + len > pool.cap) {
                flags[1] = 1u;  // pool exhausted: host grows it and reruns
                poff[j] = 0;
                plen[j] = 0;
            } else {
                kway_merge(in, pool.key + at, pool.cnt + at, &flags[0]);
                poff[j] = at;
                plen[j] = len;
            }
        }
        // Kahn: release predecessors; aggregate the pushes per warp
        std::uint64_t r0 = 0;
        std::uint32_t rn = 0;
        if (valid) {
            r0 = roff[j];
            rn = rcnt[j];
        }
        for (;;) {
            // process releases in rounds of at most 4 per lane
            std::uint32_t rel[4];
            unsigned nrel = 0;
            while (rn && nrel < 4) {
                const std::uint32_t p = rsrc[r0++];
                --rn;
                if (atomicSub(&pending[p], 1u) == 1u) rel[nrel++] = p;
            }
            const unsigned long long q = warp_reserve(next_count, nrel);
            for (unsigned k = 0; k < nrel; ++k) next[q + k] = rel[k];
            if (!__any_sync(0xffffffffu, rn != 0)) break;
        }
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

}  // namespace

// ---------------------------------------------------------------------------------
// host wrappers
// ---------------------------------------------------------------------------------

int launch_mark_sources(const std::uint8_t* codes, const Dims& d, const void* src, std::uint64_t n,
                        int id_width, std::uint8_t* marked, std::uint32_t* nodes,
                        std::uint32_t* nid, unsigned int* bad, cudaStream_t s, int num_sms) {
    if (n == 0) return MSC3D_OK;
    if (id_width == 4)
        k_mark_sources<std::uint32_t><<<grid_for(n, num_sms), kThreads, 0, s>>>(
            codes, d, static_cast<const std::uint32_t*>(src), n, marked, nodes, nid, bad);
    else
        k_mark_sources<std::uint64_t><<<grid_for(n, num_sms), kThreads, 0, s>>>(
            codes, d, static_cast<const std::uint64_t*>(src), n, marked, nodes, nid, bad);
    count_launch();
    MSC3D_CUDA_TRY(cudaGetLastError());
    return MSC3D_OK;
}

int launch_bfs_level(const std::uint8_t* codes, const Dims& d, std::uint8_t* marked,
                     std::uint32_t* nodes, std::uint64_t begin, std::uint64_t end,
                     unsigned long long* tail, std::uint32_t* nid, cudaStream_t s, int num_sms) {
    if (end <= begin) return MSC3D_OK;
    k_bfs_level<<<grid_for(end - begin, num_sms, 32), kThreads, 0, s>>>(codes, d, marked, nodes,
                                                                        begin, end, tail, nid);
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

int launch_node_succ(const std::uint8_t* codes, const Dims& d, const std::uint32_t* nodes,
                     std::uint64_t m, const std::uint32_t* nid, const std::uint32_t* tmap,
                     std::uint32_t* succ, std::uint8_t* outdeg, cudaStream_t s, int num_sms) {
    if (m == 0) return MSC3D_OK;
    k_node_succ<<<grid_for(m, num_sms), kThreads, 0, s>>>(codes, d, nodes, m, nid, tmap, succ, outdeg);
    count_launch();
    MSC3D_CUDA_TRY(cudaGetLastError());
    return MSC3D_OK;
}

int launch_chain_ptr(const std::uint32_t* succ, const std::uint8_t* outdeg, std::uint64_t m,
                     std::uint64_t n_src, std::uint32_t* ptr, cudaStream_t s, int num_sms) {
    if (m == 0) return MSC3D_OK;
    k_chain_ptr<<<grid_for(m, num_sms), kThreads, 0, s>>>(succ, outdeg, m, n_src, ptr);
    count_launch();
    MSC3D_CUDA_TRY(cudaGetLastError());
    return MSC3D_OK;
}

int launch_junction_flags(const std::uint8_t* outdeg, std::uint64_t m, std::uint64_t n_src,
                          std::uint32_t* flag, cudaStream_t s, int num_sms) {
    if (m == 0) return MSC3D_OK;
    k_junction_flags<<<grid_for(m, num_sms), kThreads, 0, s>>>(outdeg, m, n_src, flag);
    count_launch();
    MSC3D_CUDA_TRY(cudaGetLastError());
    return MSC3D_OK;
}

int launch_junction_write(const std::uint32_t* flag, const std::uint64_t* off, std::uint64_t m,
                          std::uint32_t* jlist, std::uint32_t* jidx, cudaStream_t s, int num_sms) {
    if (m == 0) return MSC3D_OK;
    k_junction_write<<<grid_for(m, num_sms), kThreads, 0, s>>>(flag, off, m, jlist, jidx);
    count_launch();
    MSC3D_CUDA_TRY(cudaGetLastError());
    return MSC3D_OK;
}

int launch_origin_dests(const std::uint32_t* jlist, std::uint64_t n, const std::uint32_t* succ,
                        const std::uint8_t* outdeg, const std::uint32_t* stop,
                        const std::uint32_t* jidx, std::uint32_t* dest, std::uint32_t* pending,
                        std::uint32_t* indeg, cudaStream_t s, int num_sms) {
    if (n == 0) return MSC3D_OK;
    k_origin_dests<<<grid_for(n, num_sms), kThreads, 0, s>>>(jlist, n, succ, outdeg, stop, jidx,
                                                            dest, pending, indeg);
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

int launch_kahn_level(const std::uint32_t* frontier, std::uint64_t nf, const std::uint32_t* dest,
                      std::uint64_t* poff, std::uint32_t* plen, std::uint32_t* pkey,
                      std::uint64_t* pcnt, unsigned long long* ptop, std::uint64_t pcap,
                      const std::uint64_t* roff, const std::uint32_t* rcnt, const std::uint32_t* rsrc,
                      std::uint32_t* pending, std::uint32_t* next, unsigned long long* next_count,
                      unsigned int* flags, cudaStream_t s, int num_sms) {
    if (nf == 0) return MSC3D_OK;
    Pool pool{pkey, pcnt, ptop, pcap};
    k_kahn_level<<<grid_for(nf, num_sms, 32), kThreads, 0, s>>>(frontier, nf, dest, poff, plen, pool,
                                                              roff, rcnt, rsrc, pending, next,
                                                              next_count, flags);
    count_launch();
    MSC3D_CUDA_TRY(cudaGetLastError());
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

// Extremum forests, root finding and saddle-extremum arcs
// (proj/src/extrema.cpp:43-155), plus the id remaps the assembly needs
// (proj/src/msc.cpp:110-145).
//
//  * k_forest0 / k_forest3: build_forest from pair codes (the compute() pipeline
//    gets the same parents for free from the gradient kernel).
//  * k_double: one synchronous pointer-doubling round next[i] = label[label[i]]
//    (extrema.cpp:79-101) -- bit-exact labels AND round count for find_roots.
//  * k_tile_roots + k_jump_all + k_resolve_exits: in-place pointer jumping (same
//    fixpoint, fewer passes) for the compute() pipeline, where the round count is
//    not observable: box-local doubling on smooth fields, then both forests' global
//    jumping in one cooperative launch.
//  * se kernels: per saddle, the roots of its two descending (1-saddle) or
//    ascending (2-saddle) walks, merged into multiplicity-2 arcs when equal.
#include <cooperative_groups.h>

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

// The other endpoint of a vertex's paired edge is the vertex one stride away along the
// code's axis (extrema.cpp:51-57); a cube's paired quad leads to the cube one stride
// away along its axis, if that cube exists (extrema.cpp:68-75) -- index arithmetic on
// the dense ids, no lattice coordinates beyond the vertex / cube position.
__global__ void k_forest0(const std::uint8_t* __restrict__ codes, Dims d,
                          std::uint32_t* __restrict__ parent) {
    const std::uint64_t vstep[3] = {1, static_cast<std::uint64_t>(d.nx), static_cast<std::uint64_t>(d.nx * d.ny)};
    GRID_STRIDE(i, d.n_verts) {
        const std::uint8_t k = codes[vertex_cell(d, i)];
        if (k == kCritical) {
            parent[i] = static_cast<std::uint32_t>(i);
            continue;
        }
        const int dir = k - kCofacetBase, axis = dir >> 1;  // a vertex pairs with a cofacet edge
        parent[i] = static_cast<std::uint32_t>((dir & 1) ? i + vstep[axis] : i - vstep[axis]);
    }
}

__global__ void k_forest3(const std::uint8_t* __restrict__ codes, Dims d,
                          std::uint32_t* __restrict__ parent) {
    const std::uint64_t mx = d.nx - 1, my = d.ny - 1, mz = d.nz - 1;
    const std::uint64_t cstep[3] = {1, mx, mx * my};
    GRID_STRIDE(i, d.n_cubes) {
        const std::uint64_t r = d.fmx.div(i), x = i - r * mx, z = d.fmy.div(r), y = r - z * my;
        const std::uint8_t k = codes[pack(d, 2 * x + 1, 2 * y + 1, 2 * z + 1)];
        if (k == kCritical) {
            parent[i] = static_cast<std::uint32_t>(i);
            continue;
        }
        const int dir = k - kFacetBase, axis = dir >> 1;  // a cube pairs with a facet quad
        const std::uint64_t coord = axis == 0 ? x : (axis == 1 ? y : z);
        const std::uint64_t ext = axis == 0 ? mx : (axis == 1 ? my : mz);
        const bool inside = (dir & 1) ? coord + 1 < ext : coord > 0;
        parent[i] = static_cast<std::uint32_t>(!inside ? i : ((dir & 1) ? i + cstep[axis] : i - cstep[axis]));
    }
}

__global__ void k_double(const std::uint32_t* __restrict__ in, std::uint32_t* __restrict__ out,
                         std::uint64_t n, unsigned int* changed) {
    bool any = false;
    GRID_STRIDE(i, n) {
        const std::uint32_t l = in[i];
        const std::uint32_t nl = in[l];
        out[i] = nl;
        any |= nl != l;
    }
    if (__any_sync(0xffffffffu, any) && (threadIdx.x & 31) == 0) *changed = 1u;
}

// Tile-local pre-resolution of a forest whose parents are lattice neighbours (both
// extremum forests: a vertex's parent is the other end of its paired edge, a cube's the
// cube across its paired quad).  One block per kTRx x kTRy x kTRz box of the forest's
// grid: the parents are read into shared memory as box-local links (root, neighbour
// inside the box, or exit = a neighbour outside it), resolved there by pointer doubling
// (shared-memory latency, not L2), and every item is written back pointing at its root
// or at the first item outside the box on its path.  The global jumping that follows
// (k_jump_all) then chases box-to-box hops: on smooth fields, where descending chains
// run for hundreds of cells, that is a factor ~16 fewer dependent random loads.
constexpr int kTRx = 32, kTRy = 16, kTRz = 16, kTRn = kTRx * kTRy * kTRz;
constexpr std::uint32_t kExit = 0x80000000u;  // link flag: the chain leaves the box

__global__ void __launch_bounds__(1024)
k_tile_roots(std::uint32_t* __restrict__ p, std::uint32_t gx, std::uint32_t gy, std::uint32_t gz,
             unsigned int* __restrict__ skip, std::uint64_t kofs, unsigned int* __restrict__ cycle) {
    // box-local link, or kExit | s: s is the box item whose parent leaves the box (its
    // parent in p never changes below -- it is s's own answer -- so it is re-read there)
    __shared__ std::uint32_t lk[kTRn];
    const std::uint32_t bx = (gx + kTRx - 1) / kTRx, by = (gy + kTRy - 1) / kTRy;
    const std::uint32_t tb = blockIdx.x;
    const std::uint32_t ox = (tb % bx) * kTRx, oy = ((tb / bx) % by) * kTRy, oz = (tb / (bx * by)) * kTRz;
    const std::uint64_t sy = gx, sz = static_cast<std::uint64_t>(gx) * gy;
    // 1. links
    for (int t = threadIdx.x; t < kTRn; t += blockDim.x) {
        const int lx = t % kTRx, ly = (t / kTRx) % kTRy, lz = t / (kTRx * kTRy);
        const std::uint32_t x = ox + lx, y = oy + ly, z = oz + lz;
        if (x >= gx || y >= gy || z >= gz) {
            lk[t] = static_cast<std::uint32_t>(t);  // padding: a root no one points at
            continue;
        }
        const std::uint64_t i = x + sy * y + sz * z;
        const std::uint32_t j = p[i];
        const std::int64_t dlt = static_cast<std::int64_t>(j) - static_cast<std::int64_t>(i);
        int nx = lx, ny = ly, nz = lz;
        if (dlt == 1) ++nx;
        else if (dlt == -1) --nx;
        else if (dlt == static_cast<std::int64_t>(sy)) ++ny;
        else if (dlt == -static_cast<std::int64_t>(sy)) --ny;
        else if (dlt == static_cast<std::int64_t>(sz)) ++nz;
        else if (dlt == -static_cast<std::int64_t>(sz)) --nz;
        else if (dlt != 0) nx = -1;  // not a lattice neighbour (cannot happen): leave it to the global pass
        const bool inside = nx >= 0 && nx < kTRx && ny >= 0 && ny < kTRy && nz >= 0 && nz < kTRz &&
                            ox + nx < gx && oy + ny < gy && oz + nz < gz;
        lk[t] = inside ? static_cast<std::uint32_t>(nx + kTRx * (ny + kTRy * nz)) : (kExit | static_cast<std::uint32_t>(t));
        if (!inside && skip) {  // j is an exit target: one of the items the global pass must resolve
            const std::uint64_t k = kofs + j;
            atomicAnd(&skip[k >> 5], ~(1u << (k & 31)));
        }
    }
    __syncthreads();
    // 2. pointer doubling inside the box until nothing changes (chains in a box are at
    //    most kTRn long): each round reads every link's link, then (after a barrier)
    //    writes them -- no thread reads a word another one is writing.  (1024 threads:
    //    kTRn / 1024 items each, kept in registers between the two halves.)
    constexpr int kMaxRounds = 16;  // 2^14 > kTRn: a chain inside the box is resolved by then
    constexpr int kPer = kTRn / 1024;
    int round = 0;
    for (; round < kMaxRounds; ++round) {
        bool ch = false;
        std::uint32_t nv[kPer];
        unsigned upd = 0;
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            const std::uint32_t l = lk[threadIdx.x + 1024 * k];
            nv[k] = l;
            if (l & kExit) continue;
            const std::uint32_t l2 = lk[l];
            if (l2 != l) {
                nv[k] = l2;
                upd |= 1u << k;
            }
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kPer; ++k)
            if ((upd >> k) & 1u) lk[threadIdx.x + 1024 * k] = nv[k];
        ch = upd != 0;
        if (!__syncthreads_or(ch)) break;  // (also the round's barrier)
    }
    if (round == kMaxRounds && threadIdx.x == 0) *cycle = 1u;  // a closed path in the box: invalid gradient
    // 3. back: the root's or the exit's global index
    for (int t = threadIdx.x; t < kTRn; t += blockDim.x) {
        const int lx = t % kTRx, ly = (t / kTRx) % kTRy, lz = t / (kTRx * kTRy);
        const std::uint32_t x = ox + lx, y = oy + ly, z = oz + lz;
        if (x >= gx || y >= gy || z >= gz) continue;
        const std::uint32_t l = lk[t];
        std::uint32_t g;
        if (l & kExit) {
            const std::uint32_t e = l & ~kExit;
            const int ex_ = static_cast<int>(e % kTRx), ey_ = static_cast<int>((e / kTRx) % kTRy),
                      ez_ = static_cast<int>(e / (kTRx * kTRy));
            g = p[(ox + ex_) + sy * (oy + ey_) + sz * (oz + ez_)];
        } else {
            const int rx = static_cast<int>(l % kTRx), ry = static_cast<int>((l / kTRx) % kTRy),
                      rz = static_cast<int>(l / (kTRx * kTRy));
            g = static_cast<std::uint32_t>((ox + rx) + sy * (oy + ry) + sz * (oz + rz));
        }
        p[x + sy * y + sz * z] = g;
    }
}

// Both forests' roots in one cooperative launch: rounds of in-place jumping over the
// concatenated index space of parent0 and parent3, a grid barrier per round and a
// rotating "changed" flag -- no host round trip per round.  conv: one bit per item,
// set once the item points at a root (final: roots never move); rounds after the
// first read the bitmap word of 32 items (L2-resident) and skip converged items
// instead of re-reading their parents' random lines.  flags[0..2] zeroed by the
// caller; rounds_out[0] = rounds run.
__global__ void k_jump_all(std::uint32_t* __restrict__ p0, std::uint64_t n0, std::uint32_t* __restrict__ p3,
                           std::uint64_t n3, unsigned int* __restrict__ conv, unsigned int* flags,
                           unsigned long long* rounds_out, int masked) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    const std::uint64_t n = n0 + n3;
    const std::uint64_t stride = static_cast<std::uint64_t>(gridDim.x) * blockDim.x;
    const std::uint64_t wstart = (blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x) & ~31ull;
    const unsigned lane = threadIdx.x & 31u;
    int round = 0;
    for (;; ++round) {
        if (grid.thread_rank() == 0) flags[(round + 1) % 3] = 0u;
        bool any = false;
        for (std::uint64_t base = wstart; base < n; base += stride) {
            const std::uint64_t k = base + lane;
            const unsigned word = (round || masked) ? conv[base >> 5] : 0u;
            bool now = false;
            if (k < n && !((word >> lane) & 1u)) {
                std::uint32_t* p = k < n0 ? p0 : p3;
                const std::uint64_t i = k < n0 ? k : k - n0;
                const std::uint32_t l = p[i];
                std::uint32_t nl = p[l];
                if (nl != l) {
#pragma unroll
                    for (int s = 0; s < 15; ++s) {
                        const std::uint32_t nn = p[nl];
                        if (nn == nl) {
                            now = true;
                            break;
                        }
                        nl = nn;
                    }
                    p[i] = nl;
                    any = true;
                } else {
                    now = true;
                }
            }
            const unsigned bits = __ballot_sync(0xffffffffu, now);
            if (lane == 0 && (bits || (!round && !masked))) conv[base >> 5] = word | bits;
        }
        if (__any_sync(0xffffffffu, any) && lane == 0) atomicOr(&flags[round % 3], 1u);
        grid.sync();
        if (*reinterpret_cast<volatile unsigned int*>(&flags[round % 3]) == 0u) break;
        if (round > 64) break;  // a cycle (invalid gradient): reported by the caller
    }
    if (grid.thread_rank() == 0) *rounds_out = static_cast<unsigned long long>(round + 1);
}

// four labels per thread with 16-byte loads and stores (label arrays are 16-byte aligned)
__global__ void k_gather(const std::uint32_t* __restrict__ label, RankRemap remap, std::uint64_t n,
                         std::uint32_t* __restrict__ out) {
    const std::uint64_t n4 = n / 4;
    GRID_STRIDE(q, n4) {
        const uint4 l = __ldcs(reinterpret_cast<const uint4*>(label) + q);
        __stcs(reinterpret_cast<uint4*>(out) + q, make_uint4(remap(l.x), remap(l.y), remap(l.z), remap(l.w)));
    }
    const std::uint64_t t = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x;
    if (t < n - 4 * n4) out[4 * n4 + t] = remap(label[4 * n4 + t]);
}

// bit of dense(crit[k]) in a zeroed bitmap
template <typename IdT>
__global__ void k_mark_bits(const IdT* __restrict__ crit, std::uint64_t n, Dims d, int dim,
                            unsigned int* __restrict__ bits) {
    GRID_STRIDE(k, n) {
        const Coord c = unpack(d, crit[k]);
        const std::uint32_t di = dim == 0 ? vertex_dense(d, c) : cube_dense(d, c);
        atomicOr(&bits[di >> 5], 1u << (di & 31));
    }
}
__global__ void k_word_popc(const unsigned int* __restrict__ bits, std::uint64_t nwords,
                            std::uint32_t* __restrict__ cnt) {
    GRID_STRIDE(w, nwords) cnt[w] = static_cast<std::uint32_t>(__popc(bits[w]));
}
__global__ void k_pack_rank(const unsigned int* __restrict__ bits, const std::uint64_t* __restrict__ pre,
                            std::uint64_t nwords, uint2* __restrict__ rank) {
    GRID_STRIDE(w, nwords) rank[w] = make_uint2(static_cast<std::uint32_t>(pre[w]), bits[w]);
}

// API saddle_extremum_arcs: per merged saddle, the two endpoint slots as cells.
template <typename IdT>
__global__ void k_se_slots(const std::uint8_t* __restrict__ codes, Dims d,
                           const IdT* __restrict__ saddles, std::uint64_t ns,
                           const std::uint32_t* __restrict__ l0, const std::uint32_t* __restrict__ l3,
                           std::uint64_t* __restrict__ slot, std::uint32_t* __restrict__ cnt) {
    GRID_STRIDE(i, ns) {
        const std::uint64_t s = saddles[i];
        const Coord c = unpack(d, s);
        std::uint64_t a = ~0ull, b = ~0ull;
        if (cell_dim(c) == 1) {
            // endpoints in cell_vertices order: lower coordinate first (grid.cpp:61-73)
            const int axis = (c.x & 1) ? 0 : ((c.y & 1) ? 1 : 2);
            Coord lo = c, hi = c;
            if (axis == 0) { lo.x -= 1; hi.x += 1; }
            else if (axis == 1) { lo.y -= 1; hi.y += 1; }
            else { lo.z -= 1; hi.z += 1; }
            a = vertex_cell(d, l0[vertex_dense(d, lo)]);
            b = vertex_cell(d, l0[vertex_dense(d, hi)]);
        } else {
            // cofacets of the quad in cofacet order (-axis first), clipped
            const int axis = !(c.x & 1) ? 0 : (!(c.y & 1) ? 1 : 2);
            const std::int64_t coord = axis == 0 ? c.x : (axis == 1 ? c.y : c.z);
            const std::int64_t ext = axis == 0 ? d.ex : (axis == 1 ? d.ey : d.ez);
            std::uint64_t got[2];
            int ng = 0;
            for (int sgn = -1; sgn <= 1; sgn += 2) {
                const std::int64_t nc = coord + sgn;
                if (nc < 0 || nc >= ext) continue;
                Coord o = c;
                if (axis == 0) o.x = nc;
                else if (axis == 1) o.y = nc;
                else o.z = nc;
                const std::uint64_t root = cube_cell(d, l3[cube_dense(d, o)]);
                got[ng++] = codes[root] == kCritical ? root : ~0ull;
            }
            a = ng > 0 ? got[0] : ~0ull;
            b = ng > 1 ? got[1] : ~0ull;
        }
        // extrema.cpp:138-146: equal -> one arc of multiplicity 2; else min, max.
        std::uint64_t x = a < b ? a : b, y = a < b ? b : a;
        std::uint32_t n = 0;
        if (a != ~0ull && a == b) {
            slot[2 * i] = a | (1ull << 63);
            slot[2 * i + 1] = ~0ull;
            n = 1;
        } else {
            slot[2 * i] = x;
            slot[2 * i + 1] = y;
            n = (x != ~0ull) + (y != ~0ull);
        }
        cnt[i] = n;
    }
}

template <typename IdT>
__global__ void k_se_write(const IdT* __restrict__ saddles, std::uint64_t ns,
                           const std::uint64_t* __restrict__ slot, const std::uint64_t* __restrict__ off,
                           IdT* __restrict__ out_s, IdT* __restrict__ out_e,
                           std::uint32_t* __restrict__ out_m) {
    GRID_STRIDE(i, ns) {
        std::uint64_t at = off[i];
        for (int k = 0; k < 2; ++k) {
            const std::uint64_t v = slot[2 * i + k];
            if (v == ~0ull) continue;
            out_s[at] = saddles[i];
            out_e[at] = static_cast<IdT>(v & ~(1ull << 63));
            out_m[at] = (v >> 63) ? 2u : 1u;
            ++at;
        }
    }
}

}  // namespace

int launch_forest(const std::uint8_t* codes, const Dims& d, int dim, std::uint32_t* parent,
                  cudaStream_t s, int num_sms) {
    if (dim == 0)
        k_forest0<<<grid_for(d.n_verts, num_sms), kThreads, 0, s>>>(codes, d, parent);
    else if (d.n_cubes)
        k_forest3<<<grid_for(d.n_cubes, num_sms), kThreads, 0, s>>>(codes, d, parent);
    count_launch();
    MSC3D_CUDA_TRY(cudaGetLastError());
    return MSC3D_OK;
}

int launch_double_round(const std::uint32_t* in, std::uint32_t* out, std::uint64_t n,
                        unsigned int* changed, cudaStream_t s, int num_sms) {
    k_double<<<grid_for(n, num_sms), kThreads, 0, s>>>(in, out, n, changed);
    count_launch();
    MSC3D_CUDA_TRY(cudaGetLastError());
    return MSC3D_OK;
}

int launch_tile_roots(std::uint32_t* p, std::uint64_t gx, std::uint64_t gy, std::uint64_t gz, unsigned int* skip,
                      std::uint64_t kofs, unsigned int* cycle, cudaStream_t s) {
    if (gx == 0 || gy == 0 || gz == 0) return MSC3D_OK;
    const std::uint64_t tiles = ((gx + kTRx - 1) / kTRx) * ((gy + kTRy - 1) / kTRy) * ((gz + kTRz - 1) / kTRz);
    if (tiles > 0x7fffffffull) return MSC3D_ERR_INVALID;
    k_tile_roots<<<static_cast<unsigned>(tiles), 1024 /* kPer */, 0, s>>>(p, static_cast<std::uint32_t>(gx),
                                                               static_cast<std::uint32_t>(gy),
                                                               static_cast<std::uint32_t>(gz), skip, kofs, cycle);
    count_launch();
    MSC3D_CUDA_TRY(cudaGetLastError());
    return MSC3D_OK;
}

// After the tile pass: every item points at its root or at an exit target, and the
// exit targets (resolved by the masked global pass) point at their roots.
// Four items per thread: one 16-byte load of their pointers, the four gathers in flight
// together, a 16-byte store only when something changed (items whose box root is a
// real root are final already).  Arrays are 16-byte aligned; the < 4 tail items of
// each array go one by one.
__global__ void k_resolve_exits(std::uint32_t* __restrict__ p, std::uint64_t n) {
    const std::uint64_t n4 = n / 4;
    uint4* p4 = reinterpret_cast<uint4*>(p);
    GRID_STRIDE(k, n4) {
        const uint4 v = p4[k];
        const uint4 r = make_uint4(p[v.x], p[v.y], p[v.z], p[v.w]);
        if (r.x != v.x || r.y != v.y || r.z != v.z || r.w != v.w) p4[k] = r;
    }
    const std::uint64_t t = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x;
    if (t < n - 4 * n4) p[4 * n4 + t] = p[p[4 * n4 + t]];
}

int launch_resolve_exits(std::uint32_t* p0, std::uint64_t n0, std::uint32_t* p3, std::uint64_t n3, cudaStream_t s,
                         int num_sms) {
    if (n0) k_resolve_exits<<<grid_for((n0 + 3) / 4, num_sms), kThreads, 0, s>>>(p0, n0);
    if (n3) k_resolve_exits<<<grid_for((n3 + 3) / 4, num_sms), kThreads, 0, s>>>(p3, n3);
    count_launch(2);
    MSC3D_CUDA_TRY(cudaGetLastError());
    return MSC3D_OK;
}

int launch_jump_all(std::uint32_t* p0, std::uint64_t n0, std::uint32_t* p3, std::uint64_t n3, unsigned int* conv,
                    unsigned int* flags, unsigned long long* rounds, cudaStream_t s, int num_sms, int masked) {
    if (n0 + n3 == 0) return MSC3D_OK;
    int per_sm = 0;
    MSC3D_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_jump_all, kThreads, 0));
    if (per_sm <= 0) return MSC3D_ERR_CUDA;
    const unsigned grid = static_cast<unsigned>(std::min<std::uint64_t>(
        static_cast<std::uint64_t>(per_sm) * num_sms, std::max<std::uint64_t>(1, (n0 + n3 + kThreads - 1) / kThreads)));
    void* args[] = {&p0, &n0, &p3, &n3, &conv, &flags, &rounds, &masked};
    MSC3D_CUDA_TRY(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k_jump_all), dim3(grid), dim3(kThreads),
                                               args, 0, s));
    count_launch();
    return MSC3D_OK;
}

int launch_rank_map(const void* crit, std::uint64_t n, int id_width, const Dims& d, int dim,
                    unsigned int* bits, std::uint32_t* cnt, std::uint64_t* pre, void* rank, std::uint64_t nwords,
                    Workspace& ws, std::uint64_t* d_total, cudaStream_t s, int num_sms) {
    if (nwords == 0) return MSC3D_OK;
    MSC3D_CUDA_TRY(cudaMemsetAsync(bits, 0, nwords * 4, s));
    if (n) {
        if (id_width == 4)
            k_mark_bits<std::uint32_t><<<grid_for(n, num_sms), kThreads, 0, s>>>(
                static_cast<const std::uint32_t*>(crit), n, d, dim, bits);
        else
            k_mark_bits<std::uint64_t><<<grid_for(n, num_sms), kThreads, 0, s>>>(
                static_cast<const std::uint64_t*>(crit), n, d, dim, bits);
        count_launch();
    }
    k_word_popc<<<grid_for(nwords, num_sms), kThreads, 0, s>>>(bits, nwords, cnt);
    count_launch();
    int rc = scan_u32(cnt, nwords, pre, d_total, ws, s);
    if (rc != MSC3D_OK) return rc;
    k_pack_rank<<<grid_for(nwords, num_sms), kThreads, 0, s>>>(bits, pre, nwords, static_cast<uint2*>(rank));
    count_launch();
    MSC3D_CUDA_TRY(cudaGetLastError());
    return MSC3D_OK;
}

int launch_gather(const std::uint32_t* label, RankRemap remap, std::uint64_t n,
                  std::uint32_t* out, cudaStream_t s, int num_sms) {
    if (n == 0) return MSC3D_OK;
    k_gather<<<grid_for(n / 4 + 1, num_sms), kThreads, 0, s>>>(label, remap, n, out);
    count_launch();
    MSC3D_CUDA_TRY(cudaGetLastError());
    return MSC3D_OK;
}

int launch_se_slots(const std::uint8_t* codes, const Dims& d, const void* saddles,
                    std::uint64_t ns, int id_width, const std::uint32_t* l0,
                    const std::uint32_t* l3, std::uint64_t* slot, std::uint32_t* cnt,
                    cudaStream_t s, int num_sms) {
    if (ns == 0) return MSC3D_OK;
    if (id_width == 4)
        k_se_slots<std::uint32_t><<<grid_for(ns, num_sms), kThreads, 0, s>>>(
            codes, d, static_cast<const std::uint32_t*>(saddles), ns, l0, l3, slot, cnt);
    else
        k_se_slots<std::uint64_t><<<grid_for(ns, num_sms), kThreads, 0, s>>>(
            codes, d, static_cast<const std::uint64_t*>(saddles), ns, l0, l3, slot, cnt);
    count_launch();
    MSC3D_CUDA_TRY(cudaGetLastError());
    return MSC3D_OK;
}

int launch_se_write(const void* saddles, std::uint64_t ns, int id_width,
                    const std::uint64_t* slot, const std::uint64_t* off, void* out_s, void* out_e,
                    std::uint32_t* out_m, cudaStream_t s, int num_sms) {
    if (ns == 0) return MSC3D_OK;
    if (id_width == 4)
        k_se_write<std::uint32_t><<<grid_for(ns, num_sms), kThreads, 0, s>>>(
            static_cast<const std::uint32_t*>(saddles), ns, slot, off,
            static_cast<std::uint32_t*>(out_s), static_cast<std::uint32_t*>(out_e), out_m);
    else
        k_se_write<std::uint64_t><<<grid_for(ns, num_sms), kThreads, 0, s>>>(
            static_cast<const std::uint64_t*>(saddles), ns, slot, off,
            static_cast<std::uint64_t*>(out_s), static_cast<std::uint64_t*>(out_e), out_m);
    count_launch();
    MSC3D_CUDA_TRY(cudaGetLastError());
    return MSC3D_OK;
}

}  // namespace msc3d_dev

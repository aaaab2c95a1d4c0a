// The saddle-saddle DAG on the device, built around a per-edge successor table.
//
// Successor table.  The DAG of the reference (saddle_graph.cpp:10-24) has the 1-cells
// as nodes; a 1-cell e has at most four cofacet quads q (two even axes b, two signs
// s, in cofacet order), and q contributes: a terminal 2-saddle (q critical), nothing
// (q paired with a cube, or with e itself, or outside the box), or the edge q is
// paired with -- which is one of three edges: the one parallel to e across q
// ("straight") or one of the two edges of q along b ("turn" towards -a / +a, a the
// odd axis of e).  That is 5 states = 3 bits per cofacet position, 12 bits per edge,
// plus one bit "e is critical".  k_succ_table derives the 16-bit word of every edge
// from the pair codes in one pass; afterwards every DAG step is ONE 2-byte load and
// integer arithmetic on the dense edge index de = 3 * (lower vertex) + axis -- no
// lattice-coordinate divisions, no per-step byte gathers from the 1 GB code array.
//
// Reachability (mark_reachable, saddle_graph.cpp:26-86): level-synchronous BFS in
// one cooperative kernel (a grid barrier per level), 32 frontier nodes per warp
// iteration, claims by atomic test-and-set in the visited bitmap (1 bit per dense
// edge, L2-resident), one warp-aggregated reservation per iteration for the next
// frontier.  (Depth-first / chain-following variants were measured and lose: a
// long V-path walked by one thread costs more than the BFS levels that reach the
// same nodes in parallel.)
//
// Junctions (saddle_graph.cpp:126-133) = visited, non-critical edges with > 1
// successor: a bitmap, ranked by per-word popcount prefix sums (rank(de) =
// woff[de/32] + popc(jbits[de/32] & below)), so no 1.6 GB id-map is scattered.
//
// Counting (path_matrix.cpp:188-219).  Every junction / 1-saddle branch is walked
// to its end (k_walk).  Each junction j then needs P(j), the sorted sparse vector
// of path counts to 2-saddles, P(j) = sum over branches of P(dest): Kahn's
// algorithm over the junction graph -- a cooperative kernel runs round 0 over the
// nodes without pending children (in index order, from the rewrite) and the big early
// rounds over the frontier of nodes whose last child finished in the previous round;
// an asynchronous kernel finishes the rest without rounds (k_count_async: a node is
// merged as soon as its last child is).  P(j) with <= 2 entries is stored inline in a 32-byte record,
// longer ones in a pool (64 arenas, one reservation per warp).  1-saddles are the
// roots: they only record their merged length; a final pass writes the sorted
// (1-saddle, 2-saddle, count) output.  Counts are exact u64 with sticky overflow.
#include <cooperative_groups.h>

#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace msc3d_dev {

namespace {

constexpr int kThreads = 256;
constexpr std::uint32_t kTerm = 0x80000000u;
constexpr std::uint32_t kNone = 0xffffffffu;
constexpr std::uint32_t kSuccCrit = 1u << 12;
constexpr std::uint32_t kFieldLow = 0x249u;  // lowest bit of each 3-bit field
constexpr int kArenas = 64;
constexpr std::uint64_t kBadOff = ~0ull;
// dead-junction path bound Z (see JRec): f32 bits in a record's kind word
constexpr float kZLimit = 18446744073709551616.0f;  // 2^64
__device__ __forceinline__ std::uint32_t zword(float z) { return __float_as_uint(z) << 1; }
__device__ __forceinline__ float zof(std::uint32_t kind) { return __uint_as_float(kind >> 1); }

// One item per thread, blocks in id order: the resident blocks then sweep the id
// space as a compact wavefront, so the random accesses of neighbouring items (which
// are spatial neighbours) share the L2.  (A capped grid with a grid-stride loop lets
// blocks drift apart across the whole volume and defeats the L2.)
inline unsigned grid_full(std::uint64_t n) {
    return static_cast<unsigned>(std::max<std::uint64_t>(1, (n + kThreads - 1) / kThreads));
}

inline unsigned grid_for(std::uint64_t n, int num_sms, int per_sm = 16) {
    const std::uint64_t need = (n + kThreads - 1) / kThreads;
    return static_cast<unsigned>(std::max<std::uint64_t>(
        1, std::min<std::uint64_t>(need, static_cast<std::uint64_t>(num_sms) * per_sm)));
}

// Vertex strides as u32 (dense edge ids are < 2^32 for every grid this path takes).
struct EGrid {
    std::uint32_t sy, sz;  // nx, nx*ny
    __device__ __forceinline__ std::uint32_t st(int axis) const {
        return axis == 0 ? 1u : (axis == 1 ? sy : sz);
    }
};

// Device clock in ns, for per-round timelines (stats arrays).
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
constexpr int kTimeline = 256;

__device__ __forceinline__ int other_axis(int a, int k) { return a == 0 ? 1 + k : (a == 1 ? 2 * k : k); }

__device__ __forceinline__ std::uint32_t n_succ(std::uint32_t s) {
    return __popc((s | (s >> 1) | (s >> 2)) & kFieldLow);
}

struct EdgeRef {
    std::uint32_t v;  // lower vertex
    int a;            // odd axis
    __device__ __forceinline__ explicit EdgeRef(std::uint32_t de) {
        v = __umulhi(de, 0xAAAAAAABu) >> 1;
        a = static_cast<int>(de - 3u * v);
    }
};

// Successor edge at cofacet position p (0..3) with field f in {2, 3, 4}.
__device__ __forceinline__ std::uint32_t succ_edge(const EdgeRef& e, std::uint32_t de, int p,
                                                   std::uint32_t f, const EGrid& g) {
    const int b = other_axis(e.a, p >> 1);
    const std::uint32_t sb = g.st(b);
    const bool neg = !(p & 1);
    if (f == 2) return neg ? de - 3u * sb : de + 3u * sb;
    std::uint32_t lv = neg ? e.v - sb : e.v;
    if (f == 4) lv += g.st(e.a);
    return 3u * lv + static_cast<std::uint32_t>(b);
}
// Dense index 3 * (lower vertex) + normal axis of the terminal quad at position p.
__device__ __forceinline__ std::uint32_t term_quad(const EdgeRef& e, int p, const EGrid& g) {
    const int b = other_axis(e.a, p >> 1);
    const std::uint32_t lv = (p & 1) ? e.v : e.v - g.st(b);
    return 3u * lv + static_cast<std::uint32_t>(3 - e.a - b);
}

// Per-block step tables: every successor / terminal-quad index is the current dense
// edge id plus an offset that depends only on the edge axis a, the cofacet position p
// and the field value f (succ_edge / term_quad are linear in de), so a walk step is a
// table lookup and an add (u32 wrap-around is exact) instead of the axis arithmetic.
struct StepTables {
    std::uint32_t step[36];  // [(a * 4 + p) * 3 + f - 2]: successor edge offset, f in {2, 3, 4}
    std::uint32_t tq[12];    // [a * 4 + p]: terminal quad offset
    std::uint8_t nax[12];    // [a * 4 + p]: axis of a turn's successor edge (f in {3, 4})
};
__device__ __forceinline__ void fill_step_tables(StepTables& t, const EGrid& g) {
    // offsets read off a representative interior edge with the exact step functions
    const std::uint32_t v = g.sz + g.sy + 1u;
    for (int i = threadIdx.x; i < 36; i += blockDim.x) {
        const int a = i / 12, p = (i / 3) % 4;
        const std::uint32_t f = 2u + static_cast<std::uint32_t>(i % 3), de = 3u * v + static_cast<std::uint32_t>(a);
        t.step[i] = succ_edge(EdgeRef(de), de, p, f, g) - de;
    }
    for (int i = threadIdx.x; i < 12; i += blockDim.x) {
        const int a = i / 4, p = i % 4;
        const std::uint32_t de = 3u * v + static_cast<std::uint32_t>(a);
        t.tq[i] = term_quad(EdgeRef(de), p, g) - de;
        t.nax[i] = static_cast<std::uint8_t>(other_axis(a, p >> 1));
    }
}

// ---------------------------------------------------------------------------------
// successor table
// ---------------------------------------------------------------------------------
// One block per vertex row (vy, vz): the row's edges and their cofacet quads live in 8
// lattice rows around lattice row (2vy, 2vz); each field is one shared-memory table
// lookup lut[edge axis][position][quad code] (12 x 256 bytes, built per block) instead
// of decoding the pair code with branches -- the kernel was instruction-bound (142
// instructions per edge) on the decode and 64-bit index arithmetic.
__global__ void k_succ_lut(std::uint8_t* __restrict__ lut) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < 12 * 256; i += gridDim.x * blockDim.x) {
        const int a = i >> 10, p = (i >> 8) & 3, qc = i & 255;
        const int b = other_axis(a, p >> 1), h = p & 1;
        std::uint8_t f = 0;
        if (qc == kCritical) {
            f = 1;
        } else if (qc >= kFacetBase && qc < kFacetBase + 6) {
            const int dir = qc - kFacetBase, ax = dir >> 1, ps = dir & 1;
            if (ax == b) f = ps == h ? 2 : 0;  // the other way is e itself
            else f = ps ? 4 : 3;               // ax == a
        }
        lut[i] = f;
    }
}

__global__ void __launch_bounds__(256)
k_succ_table(const std::uint8_t* __restrict__ codes, Dims d, const uint4* __restrict__ g_lut,
             std::uint16_t* __restrict__ succ) {
    __shared__ uint4 lut4[12 * 256 / 16];
    for (int i = threadIdx.x; i < 12 * 256 / 16; i += blockDim.x) lut4[i] = g_lut[i];
    __syncthreads();
    const std::uint8_t* lut = reinterpret_cast<const std::uint8_t*>(lut4);
    const std::uint64_t rows = static_cast<std::uint64_t>(d.ny) * d.nz;
    const std::int64_t ex = d.ex, exy = d.exy;
    for (std::uint64_t r = blockIdx.x; r < rows; r += gridDim.x) {
        const std::int64_t vz = static_cast<std::int64_t>(d.fny.div(r));
        const std::int64_t vy = static_cast<std::int64_t>(r) - vz * d.ny;
        const bool ym = vy > 0, yp = vy < d.ny - 1, zm = vz > 0, zp = vz < d.nz - 1;
        const std::uint8_t* R00 = codes + (2 * vz * d.ey + 2 * vy) * ex;  // lattice row (2vy, 2vz)
        const std::uint8_t *Rm0 = R00 - ex, *Rp0 = R00 + ex, *R0m = R00 - exy, *R0p = R00 + exy;
        const std::uint8_t *Rpm = Rp0 - exy, *Rpp = Rp0 + exy, *Rmp = Rm0 + exy;
        std::uint16_t* out = succ + 3 * static_cast<std::uint64_t>(d.nx) * r;
        const int nx = static_cast<int>(d.nx);
        for (int vx = threadIdx.x; vx < nx; vx += blockDim.x) {
            const int x = 2 * vx;
            const bool xm = vx > 0, xp = vx < nx - 1;
            // all thirteen code bytes first (out-of-box neighbours read a valid in-row
            // byte and are masked below): one memory latency per vertex instead of a
            // chain of load -> table lookup -> next load
            const int xl = xm ? x - 1 : x, xr = xp ? x + 1 : x;
            const std::uint8_t* Rm0_ = ym ? Rm0 : R00;
            const std::uint8_t* Rp0_ = yp ? Rp0 : R00;
            const std::uint8_t* R0m_ = zm ? R0m : R00;
            const std::uint8_t* R0p_ = zp ? R0p : R00;
            const std::uint8_t* Rpm_ = (yp && zm) ? Rpm : R00;
            const std::uint8_t* Rpp_ = (yp && zp) ? Rpp : R00;
            const std::uint8_t* Rmp_ = (ym && zp) ? Rmp : R00;
            const std::uint32_t e0 = __ldg(R00 + xr), q0a = __ldg(Rm0_ + xr), q0b = __ldg(Rp0_ + xr),
                                q0c = __ldg(R0m_ + xr), q0d = __ldg(R0p_ + xr);
            const std::uint32_t e1 = __ldg(Rp0_ + x), q1a = __ldg(Rp0_ + xl), q1b = __ldg(Rp0_ + xr),
                                q1c = __ldg(Rpm_ + x), q1d = __ldg(Rpp_ + x);
            const std::uint32_t e2 = __ldg(R0p_ + x), q2a = __ldg(R0p_ + xl), q2b = __ldg(R0p_ + xr),
                                q2c = __ldg(Rmp_ + x), q2d = __ldg(Rpp_ + x);
            std::uint32_t w0 = 0, w1 = 0, w2 = 0;
            if (xp) {  // x-edge (x+1, 2vy, 2vz): quads -y, +y, -z, +z at x+1
                w0 = (e0 == kCritical ? kSuccCrit : 0u);
                if (ym) w0 |= static_cast<std::uint32_t>(lut[(0 << 8) | q0a]);
                if (yp) w0 |= static_cast<std::uint32_t>(lut[(1 << 8) | q0b]) << 3;
                if (zm) w0 |= static_cast<std::uint32_t>(lut[(2 << 8) | q0c]) << 6;
                if (zp) w0 |= static_cast<std::uint32_t>(lut[(3 << 8) | q0d]) << 9;
            }
            if (yp) {  // y-edge (x, 2vy+1, 2vz): quads -x, +x (same row), -z, +z
                w1 = (e1 == kCritical ? kSuccCrit : 0u);
                if (xm) w1 |= static_cast<std::uint32_t>(lut[(4 << 8) | q1a]);
                if (xp) w1 |= static_cast<std::uint32_t>(lut[(5 << 8) | q1b]) << 3;
                if (zm) w1 |= static_cast<std::uint32_t>(lut[(6 << 8) | q1c]) << 6;
                if (zp) w1 |= static_cast<std::uint32_t>(lut[(7 << 8) | q1d]) << 9;
            }
            if (zp) {  // z-edge (x, 2vy, 2vz+1): quads -x, +x (same row), -y, +y
                w2 = (e2 == kCritical ? kSuccCrit : 0u);
                if (xm) w2 |= static_cast<std::uint32_t>(lut[(8 << 8) | q2a]);
                if (xp) w2 |= static_cast<std::uint32_t>(lut[(9 << 8) | q2b]) << 3;
                if (ym) w2 |= static_cast<std::uint32_t>(lut[(10 << 8) | q2c]) << 6;
                if (yp) w2 |= static_cast<std::uint32_t>(lut[(11 << 8) | q2d]) << 9;
            }
            out[3 * vx] = static_cast<std::uint16_t>(w0);
            out[3 * vx + 1] = static_cast<std::uint16_t>(w1);
            out[3 * vx + 2] = static_cast<std::uint16_t>(w2);
        }
    }
}

// ---------------------------------------------------------------------------------
// reachability: rounds of chain-following traversal, one cooperative launch
// ---------------------------------------------------------------------------------
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

// Frontier appends through a per-warp shared-memory queue: one global reservation
// per block per round (flush_block) instead of one per warp iteration -- a single
// frontier counter hit by every warp of the grid serialises in the L2.  A warp
// queue that fills up mid-round is flushed on its own.
constexpr int kQCap = 256;

struct WarpQ {
    std::uint32_t item[kQCap];
    std::uint32_t n;
};

// `cap`: entries the output buffer holds; appends past it are dropped (the caller
// sees the counter exceed cap and retries with a larger buffer).
__device__ __forceinline__ void flush_warp(WarpQ& q, std::uint32_t* out, unsigned long long* ctr,
                                           unsigned long long cap = ~0ull) {
    const int lane = threadIdx.x & 31;
    const std::uint32_t n = q.n;
    unsigned long long base = 0;
    if (lane == 0 && n) base = atomicAdd(ctr, static_cast<unsigned long long>(n));
    base = __shfl_sync(0xffffffffu, base, 0);
    for (std::uint32_t k = lane; k < n; k += 32)
        if (base + k < cap) out[base + k] = q.item[k];
    __syncwarp();
    if (lane == 0) q.n = 0;
    __syncwarp();
}

// All lanes call; lane pushes the items[k] with bit k of `mask` set (k < 4).
__device__ __forceinline__ void warp_push(WarpQ& q, const std::uint32_t* items, unsigned mask, std::uint32_t* out,
                                          unsigned long long* ctr, unsigned long long cap = ~0ull) {
    const int lane = threadIdx.x & 31;
    const unsigned mine = __popc(mask);
    unsigned incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    const unsigned total = __shfl_sync(0xffffffffu, incl, 31);
    if (total == 0) return;
    if (q.n + total > kQCap) flush_warp(q, out, ctr, cap);
    std::uint32_t at = q.n + incl - mine;
#pragma unroll
    for (int k = 0; k < 4; ++k)
        if ((mask >> k) & 1u) q.item[at++] = items[k];
    __syncwarp();
    if (lane == 0) q.n += total;
    __syncwarp();
}

// All threads of the block call (before the grid barrier): one reservation for
// every warp queue of the block.
__device__ __forceinline__ void flush_block(WarpQ* qs, std::uint32_t* out, unsigned long long* ctr,
                                            unsigned long long cap = ~0ull) {
    __shared__ unsigned long long s_base[kThreads / 32 + 1];
    __syncthreads();
    const int nw = blockDim.x / 32;
    if (threadIdx.x == 0) {
        unsigned long long tot = 0;
        for (int w = 0; w < nw; ++w) {
            s_base[w] = tot;
            tot += qs[w].n;
        }
        const unsigned long long b = tot ? atomicAdd(ctr, tot) : 0ull;
        for (int w = 0; w < nw; ++w) s_base[w] += b;
    }
    __syncthreads();
    WarpQ& q = qs[threadIdx.x >> 5];
    const unsigned long long base = s_base[threadIdx.x >> 5];
    for (std::uint32_t k = threadIdx.x & 31; k < q.n; k += 32)
        if (base + k < cap) out[base + k] = q.item[k];
    __syncthreads();
    if ((threadIdx.x & 31) == 0) q.n = 0;
    __syncthreads();
}

// cnt[0] = number of (already claimed) seeds in fa; cnt[1], cnt[2] scratch.
// stats[0] = rounds, stats[1] = nodes claimed here.  Level-synchronous: one
// round per BFS level, 32 nodes per warp iteration, one reservation per iteration.
__global__ void __launch_bounds__(kThreads, 6)
k_reach(const std::uint16_t* __restrict__ succ, EGrid g, unsigned int* __restrict__ bitmap,
        std::uint32_t* __restrict__ fa, std::uint32_t* __restrict__ fb, unsigned long long* __restrict__ cnt,
        unsigned long long* __restrict__ stats, unsigned long long cap) {
    __shared__ WarpQ s_q[kThreads / 32];
    __shared__ StepTables s_tab;
    fill_step_tables(s_tab, g);
    WarpQ& wq = s_q[threadIdx.x >> 5];
    if ((threadIdx.x & 31) == 0) wq.n = 0;
    __syncthreads();
    cg::grid_group grid = cg::this_grid();
    std::uint32_t* cur = fa;
    std::uint32_t* nxt = fb;
    unsigned long long ncur = *reinterpret_cast<volatile unsigned long long*>(&cnt[0]);
    unsigned long long mine = 0;
    int round = 0;
    const std::uint64_t stride = static_cast<std::uint64_t>(gridDim.x) * blockDim.x;
    const std::uint64_t wbase = (blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x) & ~31ull;
    const int lane = threadIdx.x & 31;
    // one BFS level over cur[0, ncur): warps start at `first` and step by `step`
    auto level = [&](std::uint64_t first, std::uint64_t step, unsigned long long* next_cnt) {
        for (std::uint64_t base = first; base < ncur; base += step) {
            const std::uint64_t j = base + lane;
            std::uint32_t de[4] = {0, 0, 0, 0};
            std::uint32_t won = 0;
            if (j < ncur) {
                const std::uint32_t node = __ldcg(cur + j);
                const std::uint32_t s = succ[node];
                const int a4 = 4 * static_cast<int>(node - 3u * (__umulhi(node, 0xAAAAAAABu) >> 1));
                // claims by atomic test-and-set, the (<= 4) atomics issued back to back
                unsigned old[4];
#pragma unroll
                for (int p = 0; p < 4; ++p) {
                    const std::uint32_t f = (s >> (3 * p)) & 7u;
                    old[p] = ~0u;
                    if (f < 2) continue;
                    de[p] = node + s_tab.step[(a4 + p) * 3 + static_cast<int>(f) - 2];
                    old[p] = atomicOr(&bitmap[de[p] >> 5], 1u << (de[p] & 31));
                }
#pragma unroll
                for (int p = 0; p < 4; ++p)
                    if (!((old[p] >> (de[p] & 31)) & 1u)) won |= 1u << p;
            }
            mine += __popc(won);
            warp_push(wq, de, won, nxt, next_cnt, cap);
        }
        flush_block(s_q, nxt, next_cnt, cap);
    };
    bool overflow = false;  // a level larger than the frontier buffers (uniform: all read ncur)
    // Levels with big frontiers: the whole grid, a grid barrier per level.  Once the
    // frontier is small, block 0 finishes alone with block barriers (a level then costs
    // a few microseconds instead of a grid barrier's round trip); the other blocks exit
    // (no grid barrier follows).
    constexpr unsigned long long kSolo = 512;
    while (ncur >= kSolo) {
        unsigned long long* next_cnt = &cnt[(round + 1) % 3];
        if (grid.thread_rank() == 0) {
            cnt[(round + 2) % 3] = 0;
            if (round < kTimeline) stats[2 + round] = gtimer();
        }
        level(wbase, stride, next_cnt);
        grid.sync();
        ncur = *reinterpret_cast<volatile unsigned long long*>(next_cnt);
        ++round;
        if (ncur > cap) {
            overflow = true;
            break;
        }
        std::uint32_t* t = cur;
        cur = nxt;
        nxt = t;
    }
    if (blockIdx.x == 0 && !overflow) {
        while (ncur) {
            unsigned long long* next_cnt = &cnt[(round + 1) % 3];
            if (threadIdx.x == 0) {
                cnt[(round + 2) % 3] = 0;
                if (round < kTimeline) stats[2 + round] = gtimer();
            }
            __syncthreads();
            level(threadIdx.x & ~31u, blockDim.x, next_cnt);  // (ends with a block barrier)
            ncur = *reinterpret_cast<volatile unsigned long long*>(next_cnt);
            __syncthreads();
            ++round;
            if (ncur > cap) {
                overflow = true;
                break;
            }
            std::uint32_t* t = cur;
            cur = nxt;
            nxt = t;
        }
    }
    for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
    if ((threadIdx.x & 31) == 0 && mine) atomicAdd(&stats[1], mine);
    if (grid.thread_rank() == 0) {
        stats[0] = static_cast<unsigned long long>(round);
        if (round < kTimeline) stats[2 + round] = gtimer();
    }
    if (overflow && threadIdx.x == 0) stats[0] = ~0ull;  // (block 0 decides in the solo phase)
}

// ---------------------------------------------------------------------------------
// junction bitmap, ranks and list
// ---------------------------------------------------------------------------------
__global__ void k_junction_bits(const std::uint16_t* __restrict__ succ, const unsigned int* __restrict__ bitmap,
                                std::uint64_t nwords, unsigned int* __restrict__ jbits,
                                std::uint32_t* __restrict__ jcnt, unsigned long long* __restrict__ nodes) {
    unsigned long long mine = 0;
    for (std::uint64_t w = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x; w < nwords;
         w += static_cast<std::uint64_t>(gridDim.x) * blockDim.x) {
        const unsigned int bits = bitmap[w];
        unsigned int jb = 0;
        mine += __popc(bits);
        if (bits) {  // the word's 32 successor words as four 16-byte loads, all in flight together
            const uint4* sp = reinterpret_cast<const uint4*>(succ + 32 * w);
            const uint4 q[4] = {__ldg(sp), __ldg(sp + 1), __ldg(sp + 2), __ldg(sp + 3)};
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const std::uint32_t h[4] = {q[c].x, q[c].y, q[c].z, q[c].w};
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    const std::uint32_t s = (h[e >> 1] >> (16 * (e & 1))) & 0xffffu;
                    if (!(s & kSuccCrit) && n_succ(s) > 1) jb |= 1u << (8 * c + e);
                }
            }
            jb &= bits;
        }
        jbits[w] = jb;
        jcnt[w] = __popc(jb);
    }
    for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
    if ((threadIdx.x & 31) == 0 && mine) atomicAdd(nodes, mine);
}

// Also writes jrank[w] = (first rank of word w, junction bits of word w): a rank
// lookup in the walks is then one 8-byte load.
__global__ void k_junction_list(const unsigned int* __restrict__ jbits, std::uint64_t nwords,
                                const std::uint64_t* __restrict__ woff, std::uint32_t* __restrict__ jlist,
                                uint2* __restrict__ jrank) {
    for (std::uint64_t w = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x; w < nwords;
         w += static_cast<std::uint64_t>(gridDim.x) * blockDim.x) {
        unsigned int jb = jbits[w];
        std::uint64_t at = woff[w];
        jrank[w] = make_uint2(static_cast<std::uint32_t>(at), jb);
        while (jb) {
            const int b = __ffs(jb) - 1;
            jb &= jb - 1;
            jlist[at++] = static_cast<std::uint32_t>(32 * w + b);
        }
    }
}

__device__ __forceinline__ std::uint32_t junction_rank(const uint2* __restrict__ jrank, std::uint32_t de) {
    const uint2 r = jrank[de >> 5];
    return r.x + __popc(r.y & ((1u << (de & 31)) - 1u));
}

// ---------------------------------------------------------------------------------
// branch walks: origin -> up to 4 destinations (junction rank | kTerm|2-saddle rank | kNone)
// ---------------------------------------------------------------------------------
struct WalkCtx {
    const std::uint16_t* succ;
    EGrid g;
    const uint2* jrank;
    const std::uint32_t* tmap;  // 2-saddle rank per dense quad index, or null: trank
    const uint2* trank;         // 2-saddle rank words (term_rank)
    std::uint64_t limit;
    FastDiv fnx, fny;
    std::uint32_t nx, ny;
    std::uint64_t ex, exy;
    // Rank of the 2-saddle quad with dense index dq = 3 * (lower vertex) + normal axis
    // in the sorted 2-saddle list: its lattice cell id, then the per-32-cells rank word
    // (first rank of the word's 2-saddles, their bits) -- N/4 bytes instead of a u32
    // map over all 3V quads (12 bytes per vertex: 12.9 GB at 2^30 vertices).  The
    // map is used where it is small (one load per lookup instead of two divisions).
    __device__ __forceinline__ std::uint32_t term_rank(std::uint32_t dq) const {
        if (tmap) return __ldg(&tmap[dq]);
        const std::uint32_t v = __umulhi(dq, 0xAAAAAAABu) >> 1;
        const std::uint32_t a = dq - 3u * v;
        const std::uint32_t t = static_cast<std::uint32_t>(fnx.div(v)), vx = v - t * nx;
        const std::uint32_t vz = static_cast<std::uint32_t>(fny.div(t)), vy = t - vz * ny;
        const std::uint64_t cell = (2ull * vx + (a != 0)) + ex * (2ull * vy + (a != 1)) + exy * (2ull * vz + (a != 2));
        const uint2 r = __ldg(&trank[cell >> 5]);
        return r.x + __popc(r.y & ((1u << (cell & 31)) - 1u));
    }
};

// Walk from edge cur (axis a) to the branch's end.
__device__ __forceinline__ std::uint32_t walk_branch(const WalkCtx& c, const StepTables& t, std::uint32_t cur,
                                                     int a, unsigned int* cycle) {
    for (std::uint64_t steps = 0;; ++steps) {
        const std::uint32_t s = __ldg(&c.succ[cur]);
        const std::uint32_t present = (s | (s >> 1) | (s >> 2)) & kFieldLow;
        if (present == 0) return kNone;                       // dead end
        if (present & (present - 1)) return junction_rank(c.jrank, cur);
        const int p = (__ffs(present) - 1) / 3;
        const std::uint32_t f = (s >> (3 * p)) & 7u;
        const int ap = a * 4 + p;
        if (f == 1) return kTerm | c.term_rank(cur + t.tq[ap]);
        cur += t.step[ap * 3 + static_cast<int>(f) - 2];
        a = f == 2 ? a : t.nax[ap];
        if (steps > c.limit) {
            *cycle = 1u;  // invalid gradient (saddle_graph.cpp:173-174)
            return kNone;
        }
    }
}

// The 2-saddle rank words (WalkCtx::term_rank) from the sorted 2-saddle list: bit of
// each 2-saddle's cell id; the first list entry of a word writes the word's base rank
// (the list is sorted, so that is its own index).  Words without 2-saddles are never read.
template <typename IdT>
__global__ void k_term_rank(const IdT* __restrict__ list, std::uint64_t n, uint2* __restrict__ trank) {
    for (std::uint64_t k = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x; k < n;
         k += static_cast<std::uint64_t>(gridDim.x) * blockDim.x) {
        const std::uint64_t c = static_cast<std::uint64_t>(list[k]);
        if (k == 0 || (static_cast<std::uint64_t>(list[k - 1]) >> 5) != (c >> 5))
            trank[c >> 5].x = static_cast<std::uint32_t>(k);
        atomicOr(&trank[c >> 5].y, 1u << (c & 31));
    }
}

// Per-node parent record (32 bytes, one sector): the first kInlineParents parents,
// in the slots the rewrite's per-child counters hand out; later ones (in-degree > 8,
// rare) go to an overflow list.  (The branch destinations live in their own dense
// array, the parent count in the counters.)
constexpr int kInlineParents = 8;
// Pending-children counters are one byte per node (a node has <= 4 junction children):
// 4x less memory for the release atomics to hit (they decrement a byte inside its
// 32-bit word: the counter is >= 1 when a child releases it, so no borrow crosses into
// the neighbouring bytes).
constexpr std::uint8_t kSkip = 0xffu;  // pending0 of a contracted pass-through junction

struct alignas(16) NodeRec {
    std::uint32_t par[kInlineParents];
};
static_assert(sizeof(NodeRec) == 32, "NodeRec is one 32-byte sector");

constexpr std::uint8_t kDone = 0xfeu;  // pending0 of a node finished by the walk itself

// Decrement node q's pending byte; returns the byte's value before.
__device__ __forceinline__ std::uint32_t pending_release(std::uint8_t* pending, std::uint32_t q) {
    const std::uint32_t sh = 8u * (q & 3u);
    const std::uint32_t old = atomicSub(reinterpret_cast<unsigned int*>(pending) + (q >> 2), 1u << sh);
    return (old >> sh) & 0xffu;
}

// Leaves finished during the walk: a node whose branches all end at 2-saddles (or
// dead ends) has P = its sorted terminal keys with multiplicities.  A junction leaf
// with <= 2 distinct keys stores its inline record right here (coalesced: junctions
// are walked in index order) and sets its bit in `predone`; a 1-saddle leaf records
// its merged length.  Both get pending kDone: Kahn's round 0 skips them, and the
// rewrite drops predone children from their parents' pending counts and parent
// lists -- no atomics for the ~40% of the junction graph that are leaves.
template <typename IdT>
__global__ void __launch_bounds__(128)
k_walk(WalkCtx c, Dims d, const std::uint32_t* __restrict__ jlist, const IdT* __restrict__ srcs, std::uint64_t n,
       uint4* __restrict__ dest, std::uint8_t* __restrict__ pending, unsigned int* __restrict__ flags,
       uint4* __restrict__ rec, std::uint32_t* __restrict__ slen, unsigned int* __restrict__ predone,
       unsigned long long* __restrict__ n_predone,
       std::uint32_t* __restrict__ fwd, unsigned int* __restrict__ ptbits) {
    __shared__ StepTables s_tab;
    fill_step_tables(s_tab, c.g);
    __syncthreads();
    const std::uint64_t stride = static_cast<std::uint64_t>(gridDim.x) * blockDim.x;
    for (std::uint64_t base = (blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x) & ~31ull; base < n;
         base += stride) {
        const std::uint64_t i = base + (threadIdx.x & 31);
        bool pre = false, pt = false;
        if (i < n) {
            std::uint32_t de0;
            if (jlist) {
                de0 = jlist[i];
            } else {
                const Coord o = unpack(d, srcs[i]);
                const int a = (o.x & 1) ? 0 : ((o.y & 1) ? 1 : 2);
                de0 = 3u * static_cast<std::uint32_t>((o.x >> 1) + d.nx * ((o.y >> 1) + d.ny * (o.z >> 1))) + a;
            }
            const std::uint32_t s0 = c.succ[de0];
            const int a0 = static_cast<int>(de0 - 3u * (__umulhi(de0, 0xAAAAAAABu) >> 1));
            std::uint32_t dd[4] = {kNone, kNone, kNone, kNone};
            std::uint32_t pend = 0;
            int nd = 0;
#pragma unroll
            for (int p = 0; p < 4; ++p) {
                const std::uint32_t f = (s0 >> (3 * p)) & 7u;
                if (f == 0) continue;
                const int ap = a0 * 4 + p;
                const std::uint32_t t = f == 1 ? (kTerm | c.term_rank(de0 + s_tab.tq[ap]))
                                               : walk_branch(c, s_tab, de0 + s_tab.step[ap * 3 + static_cast<int>(f) - 2],
                                                             f == 2 ? a0 : s_tab.nax[ap], &flags[2]);
                dd[0] = nd == 0 ? t : dd[0];
                dd[1] = nd == 1 ? t : dd[1];
                dd[2] = nd == 2 ? t : dd[2];
                dd[3] = nd == 3 ? t : dd[3];
                ++nd;
                if (!(t & kTerm)) ++pend;
            }
            dest[i] = make_uint4(dd[0], dd[1], dd[2], dd[3]);
            if (pend == 0) {
                // terminal keys (kNone sorts last), sorted, runs counted
                std::uint32_t k[4] = {dd[0] & ~kTerm, dd[1] & ~kTerm, dd[2] & ~kTerm, dd[3] & ~kTerm};
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (dd[q] == kNone) k[q] = 0xffffffffu;
                auto ce = [](std::uint32_t& x, std::uint32_t& y) {
                    const std::uint32_t lo = min(x, y), hi = max(x, y);
                    x = lo;
                    y = hi;
                };
                ce(k[0], k[1]);
                ce(k[2], k[3]);
                ce(k[0], k[2]);
                ce(k[1], k[3]);
                ce(k[1], k[2]);
                std::uint32_t uk[4] = {0, 0, 0, 0}, uc[4] = {0, 0, 0, 0};
                std::uint32_t m = 0;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    if (k[q] == 0xffffffffu) continue;
                    const bool same = q > 0 && k[q] == k[q - 1];
                    if (!same) ++m;
#pragma unroll
                    for (int z = 0; z < 4; ++z)
                        if (static_cast<std::uint32_t>(z) == m - 1) {
                            uk[z] = k[q];
                            uc[z] += 1;
                        }
                }
                if (!jlist) {
                    slen[i] = m;
                    pre = true;
                } else if (m <= 2) {
                    rec[2 * i] = make_uint4(m, uk[0], uk[1], m == 0 ? zword(1.0f) : 0u);  // dead leaf: Z = 1
                    rec[2 * i + 1] = make_uint4(uc[0], 0u, uc[1], 0u);
                    pre = true;
                }
            }
            pending[i] = pre ? kDone : static_cast<std::uint8_t>(pend);
            if (fwd) {  // pass-through: one live branch, ending at a junction (P(j) = P(child))
                int live = 0;
                std::uint32_t child = kNone;
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    if (dd[b] == kNone) continue;
                    ++live;
                    if (!(dd[b] & kTerm)) child = dd[b];
                }
                pt = live == 1 && child != kNone;
                fwd[i] = pt ? child : static_cast<std::uint32_t>(i);
            }
        }
        const unsigned bits = __ballot_sync(0xffffffffu, pre);
        const unsigned ptb = __ballot_sync(0xffffffffu, pt);
        if ((threadIdx.x & 31) == 0 && predone) {
            predone[base >> 5] = bits;
            if (bits) atomicAdd(n_predone, static_cast<unsigned long long>(__popc(bits)));
        }
        if ((threadIdx.x & 31) == 0 && ptbits) ptbits[base >> 5] = ptb;
    }
}


__device__ __forceinline__ std::uint32_t warp_excl_scan(std::uint32_t v, std::uint32_t* total) {
    const int lane = threadIdx.x & 31;
    std::uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const std::uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    *total = __shfl_sync(0xffffffffu, incl, 31);
    return incl - v;
}

// Redirect every branch through fwd; contracted junctions leave the graph
// (no branches, pending kSkip).  Each branch reference takes the next parent slot of
// its destination (the atomic's old value): slots < kInlineParents are written
// into the destination's node record right here; later ones (in-degree > 9, rare)
// are queued as (destination, slot, parent) for the overflow list.
// Junctions left with no pending child are Kahn's round 0: appended to `ready` in
// index order within a block (one reservation per block; blocks run roughly in id
// order), so round 0 runs over a dense list instead of scanning every junction.
// Each thread rewrites kRwPer nodes (i, i + kThreads, ...) with every dependent step
// issued for all their branches at once (pass-through bits, then forwards, then predone
// bits, then the slot atomics back to back): the kernel is a chain of dependent random
// loads and returning atomics, so independent nodes per thread are what hides it.
constexpr int kRwPer = 2;
__global__ void __launch_bounds__(kThreads)
k_rewrite(NodeRec* __restrict__ node, uint4* __restrict__ dest, std::uint64_t nj, std::uint64_t n_nodes,
          const std::uint32_t* __restrict__ fwd, const unsigned int* __restrict__ ptbits,
          const unsigned int* __restrict__ predone, std::uint8_t* __restrict__ pending,
          std::uint32_t* __restrict__ indeg, uint4* __restrict__ ovq,
          unsigned long long* __restrict__ ovq_n, std::uint64_t ovq_cap,
          unsigned long long* __restrict__ n_skip, std::uint32_t* __restrict__ ready,
          unsigned long long* __restrict__ n_ready) {
    constexpr int NB = 4 * kRwPer;
    __shared__ unsigned s_wc[kRwPer][kThreads / 32];
    __shared__ unsigned long long s_base;
    std::uint64_t id[kRwPer];
    bool act[kRwPer], skip[kRwPer], is_ready[kRwPer];
    std::uint32_t dd[NB];
#pragma unroll
    for (int k = 0; k < kRwPer; ++k) {
        id[k] = (blockIdx.x * static_cast<std::uint64_t>(kRwPer) + k) * kThreads + threadIdx.x;
        skip[k] = id[k] < n_nodes && id[k] < nj && ((ptbits[id[k] >> 5] >> (id[k] & 31)) & 1u);
        act[k] = id[k] < n_nodes && !skip[k];
        is_ready[k] = false;
        uint4 d4 = act[k] ? dest[id[k]] : make_uint4(kTerm, kTerm, kTerm, kTerm);
        dd[4 * k] = d4.x;
        dd[4 * k + 1] = d4.y;
        dd[4 * k + 2] = d4.z;
        dd[4 * k + 3] = d4.w;
    }
    bool live[NB], pt[NB], need[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        live[b] = !(dd[b] & kTerm);
        pt[b] = live[b] && ((__ldg(&ptbits[dd[b] >> 5]) >> (dd[b] & 31)) & 1u);
    }
    bool moved[kRwPer];
#pragma unroll
    for (int k = 0; k < kRwPer; ++k) moved[k] = false;
#pragma unroll
    for (int b = 0; b < NB; ++b)
        if (pt[b]) {
            dd[b] = __ldg(&fwd[dd[b]]);
            moved[b / 4] = true;
        }
    std::uint32_t waiting[kRwPer];  // junction children Kahn still has to finish
#pragma unroll
    for (int k = 0; k < kRwPer; ++k) waiting[k] = 0;
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        // finished in the walk: not a pending child
        need[b] = live[b] && !((__ldg(&predone[dd[b] >> 5]) >> (dd[b] & 31)) & 1u);
        waiting[b / 4] += need[b] ? 1u : 0u;
        need[b] = need[b] && id[b / 4] < nj;  // 1-saddles wait for no release: lengths come after the rounds
    }
    std::uint32_t slot[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) slot[b] = need[b] ? atomicAdd(&indeg[dd[b]], 1u) : 0u;
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        if (!need[b]) continue;
        const std::uint32_t t = dd[b];
        const std::uint32_t parent = static_cast<std::uint32_t>(id[b / 4]);
        if (slot[b] < static_cast<std::uint32_t>(kInlineParents)) {
            node[t].par[slot[b]] = parent;
        } else {
            const unsigned long long q = atomicAdd(ovq_n, 1ull);
            if (q < ovq_cap) ovq[q] = make_uint4(t, slot[b], parent, 0u);
        }
    }
#pragma unroll
    for (int k = 0; k < kRwPer; ++k) {
        if (skip[k]) pending[id[k]] = kSkip;  // (its record is never read again)
        if (!act[k]) continue;
        if (pending[id[k]] != kDone) {
            pending[id[k]] = static_cast<std::uint8_t>(waiting[k]);
            is_ready[k] = id[k] < nj && waiting[k] == 0;
        }
        if (moved[k])  // (most records are unchanged)
            dest[id[k]] = make_uint4(dd[4 * k], dd[4 * k + 1], dd[4 * k + 2], dd[4 * k + 3]);
    }
    // Kahn's round 0 = the junctions without pending children, in index order within
    // the block (one reservation per block)
    const unsigned lane = threadIdx.x & 31u, w = threadIdx.x >> 5;
    unsigned rb[kRwPer];
#pragma unroll
    for (int k = 0; k < kRwPer; ++k) {
        rb[k] = __ballot_sync(0xffffffffu, is_ready[k]);
        const unsigned sb = __ballot_sync(0xffffffffu, skip[k]);
        if (lane == 0) {
            s_wc[k][w] = __popc(rb[k]);
            if (sb) atomicAdd(n_skip, static_cast<unsigned long long>(__popc(sb)));
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned tot = 0;
        for (int k = 0; k < kRwPer; ++k)
            for (int q = 0; q < kThreads / 32; ++q) {
                const unsigned c = s_wc[k][q];
                s_wc[k][q] = tot;
                tot += c;
            }
        s_base = tot ? atomicAdd(n_ready, static_cast<unsigned long long>(tot)) : 0ull;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kRwPer; ++k)
        if (is_ready[k])
            ready[s_base + s_wc[k][w] + __popc(rb[k] & ((1u << lane) - 1u))] = static_cast<std::uint32_t>(id[k]);
}

// Overflow-list segments of the nodes with more than kInlineParents parents (~0.1%):
// allocated by an atomic cursor (their order is irrelevant), no scan over all nodes.
__global__ void k_parent_overflow(const std::uint32_t* __restrict__ indeg, std::uint64_t nj,
                                  std::uint64_t* __restrict__ ovoff, unsigned long long* __restrict__ total) {
    for (std::uint64_t j = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x; j < nj;
         j += static_cast<std::uint64_t>(gridDim.x) * blockDim.x) {
        const std::uint32_t k = indeg[j];
        if (k > static_cast<std::uint32_t>(kInlineParents))
            ovoff[j] = atomicAdd(total, static_cast<unsigned long long>(k - kInlineParents));
    }
}

__global__ void k_fill_overflow(const uint4* __restrict__ ovq, std::uint64_t n, const std::uint64_t* __restrict__ ovoff,
                                std::uint32_t* __restrict__ rsrc) {
    for (std::uint64_t k = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x; k < n;
         k += static_cast<std::uint64_t>(gridDim.x) * blockDim.x) {
        const uint4 e = ovq[k];
        rsrc[ovoff[e.x] + e.y - kInlineParents] = e.z;
    }
}

// ---------------------------------------------------------------------------------
// counting: sparse count vectors, "last child continues"
// ---------------------------------------------------------------------------------
// P(j) record, 32 bytes: kind 0 = inline (len <= 2: k0/c0, k1/c1), kind 1 = pool
// (c0 = offset of len sorted entries; offsets and capacities are multiples of 4 so
// keys load as aligned uint4 chunks and counts as uint4 pairs).
struct alignas(16) JRec {
    std::uint32_t len, k0, k1, kind;  // kind: bit 0 (0 inline, 1 pool) | zbits(Z) << 1
    std::uint64_t c0, c1;
};

// Dead-junction overflow bound (path_matrix.cpp:188-219).  The
// reference throws overflow_error when any A* entry -- the number of paths from a
// 1-saddle s to a junction j -- exceeds 2^64-1.  For a junction that reaches a
// 2-saddle t that entry is at most the final count (s, t), whose overflow the merges
// already detect; a DEAD junction (P(j) empty: it reaches no 2-saddle) is seen by no
// final count.  Every record therefore carries Z(j) = [j dead] + sum over junction
// children of Z(child) = the number of paths from j to dead junctions, so
// Z(s) = sum over dead d of A*[s, d] >= max_d A*[s, d] for a source s.  Z is an f32
// summed with round-up (an upper bound, 31 bits: positive f32 bit patterns) in the
// record's kind word; a gather whose sum reaches 2^64 raises flags[3] ("maybe"), and
// the host then decides exactly (stages.cu: dag_count).  Contracted pass-through
// junctions keep the bound: a dead one's paths continue 1:1 into its dead child.

struct PoolRef {
    std::uint32_t* key;
    std::uint64_t* cnt;
    unsigned long long* top;  // kArenas counters
    std::uint64_t arena_cap;  // multiple of 4
};

template <bool kL2, typename T>
__device__ __forceinline__ T ld(const T* p) {
    return kL2 ? __ldcg(p) : __ldg(p);
}

template <bool kL2>
__device__ __forceinline__ JRec load_rec(const JRec* r) {
    const uint4 a = ld<kL2>(reinterpret_cast<const uint4*>(r));
    const uint4 b = ld<kL2>(reinterpret_cast<const uint4*>(r) + 1);
    JRec o;
    o.len = a.x;
    o.k0 = a.y;
    o.k1 = a.z;
    o.kind = a.w;
    o.c0 = static_cast<std::uint64_t>(b.x) | (static_cast<std::uint64_t>(b.y) << 32);
    o.c1 = static_cast<std::uint64_t>(b.z) | (static_cast<std::uint64_t>(b.w) << 32);
    return o;
}

// Store P(u): inline (kind 0) or a pool reference (kind 1).
__device__ __forceinline__ void store_rec(JRec* rec, std::uint32_t u, std::uint32_t len, std::uint32_t kind,
                                          std::uint32_t k0, std::uint32_t k1, std::uint64_t c0, std::uint64_t c1) {
    uint4* dst = reinterpret_cast<uint4*>(rec + u);
    dst[0] = make_uint4(len, k0, k1, kind);
    dst[1] = make_uint4(static_cast<std::uint32_t>(c0), static_cast<std::uint32_t>(c0 >> 32),
                        static_cast<std::uint32_t>(c1), static_cast<std::uint32_t>(c1 >> 32));
}

// Up to four sorted input lists of one node.  Inside k_count they were written by
// other SMs during the same launch, so they are read through the L2 (kL2).
struct Inputs {
    std::uint32_t len[4];
    std::uint32_t k0[4], k1[4];
    std::uint64_t c0[4], c1[4];
    std::uint64_t off[4];  // kBadOff: inline
    float z;               // sum of the junction children's Z (dead-junction bound)
};

template <bool kL2>
__device__ __forceinline__ void gather(const uint4 d4, const JRec* __restrict__ rec, Inputs& in,
                                       unsigned int* __restrict__ zflag) {
    const std::uint32_t dd[4] = {d4.x, d4.y, d4.z, d4.w};
    // all child records are loaded first (unconditionally: record 0 stands in for
    // terminal / absent branches), so the up to eight loads are in flight together
    // instead of one record round trip after another
    uint4 ra[4], rb[4];
#pragma unroll
    for (int b = 0; b < 4; ++b) {
        const std::uint32_t t = dd[b];
        const bool need = t != kNone && !(t & kTerm);
        const uint4* p = reinterpret_cast<const uint4*>(rec + (need ? t : 0u));
        ra[b] = ld<kL2>(p);
        rb[b] = ld<kL2>(p + 1);
    }
    in.z = 0.0f;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
        const std::uint32_t t = dd[b];
        in.len[b] = 0;
        in.k0[b] = in.k1[b] = 0;
        in.c0[b] = in.c1[b] = 0;
        in.off[b] = kBadOff;
        if (t == kNone) continue;
        if (t & kTerm) {
            in.len[b] = 1;
            in.k0[b] = t & ~kTerm;
            in.c0[b] = 1;
        } else {
            const std::uint64_t c0 = static_cast<std::uint64_t>(rb[b].x) | (static_cast<std::uint64_t>(rb[b].y) << 32);
            in.len[b] = ra[b].x;
            in.z = __fadd_ru(in.z, zof(ra[b].w));
            if ((ra[b].w & 1u) == 0) {  // kind 0: inline
                in.k0[b] = ra[b].y;
                in.k1[b] = ra[b].z;
                in.c0[b] = c0;
                in.c1[b] = static_cast<std::uint64_t>(rb[b].z) | (static_cast<std::uint64_t>(rb[b].w) << 32);
            } else {
                in.off[b] = c0;
                if (c0 == kBadOff) in.len[b] = 0;  // pool exhausted: the host reruns
            }
        }
    }
    if (in.z >= kZLimit) *zflag = 1u;
}

__device__ __forceinline__ bool add_ovf(std::uint64_t a, std::uint64_t b, std::uint64_t* r) {
    *r = a + b;
    return *r < a;
}

// Merge the inputs straight from memory; emit(out_index, key, count) per output
// entry; returns the output length.  Used where staging does not apply (k_count_write,
// inputs larger than a warp buffer).  Keys are 2-saddle ranks (< 2^31), so
// 0xffffffff marks an exhausted list.
template <bool kL2, typename Emit>
__device__ __forceinline__ std::uint32_t merge(const Inputs& in, const PoolRef& pool, bool* ovf, Emit emit) {
    std::uint32_t pos[4] = {0, 0, 0, 0};
    std::uint32_t kk[4];
    auto key_at = [&](int b, std::uint32_t q) -> std::uint32_t {
        if (q >= in.len[b]) return 0xffffffffu;
        return in.off[b] != kBadOff ? ld<kL2>(pool.key + in.off[b] + q) : (q == 0 ? in.k0[b] : in.k1[b]);
    };
#pragma unroll
    for (int b = 0; b < 4; ++b) kk[b] = key_at(b, 0);
    std::uint32_t out = 0;
    for (;;) {
        const std::uint32_t best = min(min(kk[0], kk[1]), min(kk[2], kk[3]));
        if (best == 0xffffffffu) break;
        std::uint64_t sum = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            if (kk[b] != best) continue;
            const std::uint64_t c = in.off[b] != kBadOff ? ld<kL2>(pool.cnt + in.off[b] + pos[b])
                                                         : (pos[b] == 0 ? in.c0[b] : in.c1[b]);
            *ovf |= add_ovf(sum, c, &sum);
            ++pos[b];
            kk[b] = key_at(b, pos[b]);
        }
        emit(out, best, sum);
        ++out;
    }
    return out;
}

// ---------------------------------------------------------------------------------
// staged merges: every lane's inputs copied to a per-warp shared buffer first
// ---------------------------------------------------------------------------------
// A merge read straight from memory is a chain of dependent L2 loads (~0.5 us per
// entry); in the later rounds of Kahn's algorithm (long vectors in the smooth parts
// of the field) such chains decide the length of every round.  Instead each lane
// copies its <= 4 inputs into its slice of a per-warp shared buffer with
// independent 16-byte loads (all in flight at once), then merges from shared memory.
constexpr int kWarpCap = 1024;  // entries per warp buffer (larger inputs: direct merge)
constexpr int kWarpCapWide = 384;  // the high-occupancy configuration of the early rounds
constexpr std::uint32_t kHeavy = 48;  // total input length above which the whole warp merges the node

// A warp's slice of the dynamic shared memory: cap (key, count) entries.
struct WarpBuf {
    std::uint64_t* cnt;
    std::uint32_t* key;
    std::uint32_t cap;
};
constexpr std::size_t warp_buf_bytes(int cap) { return static_cast<std::size_t>(cap) * 12; }
__device__ __forceinline__ WarpBuf warp_buf(void* smem, std::uint32_t cap) {
    char* base = static_cast<char*>(smem) + (threadIdx.x >> 5) * warp_buf_bytes(static_cast<int>(cap));
    return WarpBuf{reinterpret_cast<std::uint64_t*>(base), reinterpret_cast<std::uint32_t*>(base + 8 * cap), cap};
}

// Slot of list b in the lane's staging area: lists start at multiples of 4 entries
// (16-byte aligned for the asynchronous copies).
__device__ __forceinline__ std::uint32_t staged_size(const Inputs& in) {
    return ((in.len[0] + 3u) & ~3u) + ((in.len[1] + 3u) & ~3u) + ((in.len[2] + 3u) & ~3u) + ((in.len[3] + 3u) & ~3u);
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Copy this lane's inputs to wb[base ...) (base a multiple of 4): pool lists by
// asynchronous 16-byte copies (no registers, all in flight at once), inline ones
// by plain stores.  The caller waits with cp_async_wait_all + __syncwarp.
template <bool kCounts>
__device__ __forceinline__ void stage(const Inputs& in, const PoolRef& pool, WarpBuf wb, std::uint32_t base) {
    std::uint32_t at = base;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
        const std::uint32_t n = in.len[b];
        if (in.off[b] == kBadOff) {
            if (n > 0) {
                wb.key[at] = in.k0[b];
                if (kCounts) wb.cnt[at] = in.c0[b];
            }
            if (n > 1) {
                wb.key[at + 1] = in.k1[b];
                if (kCounts) wb.cnt[at + 1] = in.c1[b];
            }
        } else {
            for (std::uint32_t q = 0; q < n; q += 4) cp_async16(&wb.key[at + q], pool.key + in.off[b] + q);
            if (kCounts)
                for (std::uint32_t q = 0; q < n; q += 2) cp_async16(&wb.cnt[at + q], pool.cnt + in.off[b] + q);
        }
        at += (n + 3u) & ~3u;
    }
}

// Merge the staged lists of this lane; emit(out_index, key, count).
template <bool kCounts, typename Emit>
__device__ __forceinline__ std::uint32_t merge_staged(const Inputs& in, WarpBuf wb, std::uint32_t base,
                                                      bool* ovf, Emit emit) {
    std::uint32_t pos[4], end[4], kk[4];
    std::uint32_t at = base;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
        pos[b] = at;
        end[b] = at + in.len[b];
        kk[b] = pos[b] < end[b] ? wb.key[pos[b]] : 0xffffffffu;
        at += (in.len[b] + 3u) & ~3u;
    }
    std::uint32_t out = 0;
    for (;;) {
        const std::uint32_t best = min(min(kk[0], kk[1]), min(kk[2], kk[3]));
        if (best == 0xffffffffu) break;
        std::uint64_t sum = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            if (kk[b] != best) continue;
            if (kCounts) *ovf |= add_ovf(sum, wb.cnt[pos[b]], &sum);
            ++pos[b];
            kk[b] = pos[b] < end[b] ? wb.key[pos[b]] : 0xffffffffu;
        }
        emit(out, best, sum);
        ++out;
    }
    return out;
}

// Number of entries < x (upper == false) or <= x (upper == true) in sorted k[0, n).
__device__ __forceinline__ std::uint32_t count_below(const std::uint32_t* k, std::uint32_t n, std::uint32_t x,
                                                     bool upper) {
    std::uint32_t lo = 0, hi = n;
    while (lo < hi) {
        const std::uint32_t mid = (lo + hi) >> 1;
        if (upper ? k[mid] <= x : k[mid] < x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// Warp-cooperative merge of ONE heavy node whose inputs are staged at wb[0, S)
// (list b at st[b], lengths in.len).  Every entry goes to its stable rank in the
// union (own position + binary-search counts in the other lists, ties ordered by
// list) in the shared scratch wb[S, S + T); then runs of equal keys (<= 4 long) are
// summed and the run heads written, compacted, to the output [ok, oc).  Returns the
// output length (uniform).  All 32 lanes call; requires S + T <= kWarpCap.
__device__ __forceinline__ std::uint32_t merge_heavy(const Inputs& in, WarpBuf wb, std::uint32_t* ok,
                                                     std::uint64_t* oc, bool* ovf) {
    const int lane = threadIdx.x & 31;
    std::uint32_t st[4], S = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
        st[b] = S;
        S += (in.len[b] + 3u) & ~3u;
    }
    const std::uint32_t T = in.len[0] + in.len[1] + in.len[2] + in.len[3];
    std::uint32_t* sk = wb.key + S;
    std::uint64_t* sc = wb.cnt + S;
    for (std::uint32_t t = lane; t < T; t += 32) {
        // list and position of the t-th entry (lists concatenated without padding)
        int b = 0;
        std::uint32_t q = t;
#pragma unroll
        for (int bb = 0; bb < 3; ++bb)
            if (b == bb && q >= in.len[bb]) {
                q -= in.len[bb];
                b = bb + 1;
            }
        std::uint32_t k = 0;
        std::uint64_t c = 0;
#pragma unroll
        for (int bb = 0; bb < 4; ++bb)
            if (bb == b) {
                k = wb.key[st[bb] + q];
                c = wb.cnt[st[bb] + q];
            }
        std::uint32_t r = q;
#pragma unroll
        for (int bb = 0; bb < 4; ++bb)
            if (bb != b) r += count_below(wb.key + st[bb], in.len[bb], k, bb < b);
        sk[r] = k;
        sc[r] = c;
    }
    __syncwarp();
    std::uint32_t out = 0;
    for (std::uint32_t base = 0; base < T; base += 32) {
        const std::uint32_t t = base + lane;
        bool head = false;
        std::uint32_t k = 0;
        std::uint64_t sum = 0;
        if (t < T) {
            k = sk[t];
            head = t == 0 || sk[t - 1] != k;
            if (head) {
                sum = sc[t];
                for (std::uint32_t v = t + 1; v < T && sk[v] == k; ++v) *ovf |= add_ovf(sum, sc[v], &sum);
            }
        }
        const unsigned hm = __ballot_sync(0xffffffffu, head);
        if (head && ok) {
            const std::uint32_t o = out + __popc(hm & ((1u << lane) - 1u));
            ok[o] = k;
            oc[o] = sum;
        }
        out += __popc(hm);
    }
    __syncwarp();
    return out;
}

// Pool allocation: all 32 lanes call (len 0 for lanes that need nothing); lengths
// rounded up to multiples of 4.  Each warp carves its requests out of a private
// chunk and reserves a new chunk (one atomic) only when the current one is used up.
constexpr std::uint32_t kPoolChunk = 4096;

struct PoolChunk {
    unsigned long long base;
    std::uint32_t left;
};

__device__ __forceinline__ std::uint64_t pool_alloc(const PoolRef& pool, PoolChunk& ch, std::uint32_t len,
                                                    unsigned int* full) {
    const int lane = threadIdx.x & 31;
    const std::uint32_t want = (len + 3u) & ~3u;
    std::uint32_t incl = want;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const std::uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    const std::uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    if (total == 0) return kBadOff;
    __syncwarp();
    const std::uint32_t left = ch.left;
    __syncwarp();  // (every lane has read it before lane 0 refills the chunk)
    if (total > left) {  // warp-uniform
        if (lane == 0) {
            const std::uint32_t take = total > kPoolChunk ? total : kPoolChunk;
            const int arena = static_cast<int>(((blockIdx.x * blockDim.x + threadIdx.x) >> 5) % kArenas);
            const unsigned long long at = atomicAdd(&pool.top[arena], static_cast<unsigned long long>(take));
            if (at + take > pool.arena_cap) {
                *full = 1u;
                ch.base = kBadOff;
                ch.left = 0;
            } else {
                ch.base = static_cast<unsigned long long>(arena) * pool.arena_cap + at;
                ch.left = take;
            }
        }
        __syncwarp();
    }
    const unsigned long long base = ch.base;
    const bool ok = base != kBadOff && total <= ch.left;
    __syncwarp();
    if (lane == 0 && ok) {
        ch.base += total;
        ch.left -= total;
    }
    __syncwarp();
    if (!ok || len == 0) return kBadOff;
    return base + incl - want;
}

struct CountArgs {
    const uint4* dest;           // branch destinations per node
    const std::uint32_t* ready;  // Kahn's round 0 (from the rewrite)
    const unsigned long long* n_ready;
    const NodeRec* node;         // nj junctions, then n1 sources
    std::uint8_t* pending;       // live counters (nj + n1), one byte each
    const std::uint8_t* pending0;
    const std::uint32_t* rsrc;   // parents beyond the inline ones
    JRec* rec;
    PoolRef pool;
    std::uint32_t* slen;
    std::uint64_t nj, n1;
    std::uint32_t* fa;
    std::uint32_t* fb;
    unsigned long long* cnt;   // 3 frontier counters
    unsigned long long* stats; // [0] rounds
    unsigned long long* done;  // junctions evaluated
    unsigned int* flags;       // [0] overflow, [1] pool exhausted
    unsigned long long* diag;  // optional development diagnostics
    std::uint32_t* heavy_q;    // the round's heavy nodes
    unsigned long long* heavy_n;
    unsigned long long* heavy_head;
    const std::uint32_t* indeg;       // parents per junction (the rewrite's slot counters)
    const std::uint64_t* ovoff;       // their overflow-list offsets (in-degree > kInlineParents)
    unsigned long long switch_below;  // wide configuration: stop below this frontier size
    unsigned long long* resume;       // [0] round [1] frontier size [2] frontier buffer (0: fa, 1: fb)
};


// Release the parents of a finished junction (visible to the next round through
// the grid barrier): the first kInlineParents come with the node record, the rest
// from the overflow list; parents reaching zero pending children are appended to
// the next frontier.  All lanes call (rn = 0 for lanes without a junction).
__device__ __forceinline__ void release_parents(const CountArgs& a, WarpQ& wq, std::uint32_t rn, std::uint64_t ov,
                                                const uint4 meta, const uint4 par0, const uint4 par1,
                                                std::uint32_t* nxt, unsigned long long* next_cnt) {
    const std::uint32_t inl[kInlineParents] = {par0.x, par0.y, par0.z, par0.w, par1.x, par1.y, par1.z, par1.w};
    (void)meta;
    std::uint32_t k0 = 0;  // parents handled so far
    for (;;) {
        std::uint32_t p[4], old[4];
        const std::uint32_t m = rn - k0 < 4 ? rn - k0 : 4u;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            p[k] = kNone;
            if (k < static_cast<int>(m)) {
                const std::uint32_t q = k0 + k;
                if (q < static_cast<std::uint32_t>(kInlineParents)) {
#pragma unroll
                    for (int z = 0; z < kInlineParents; ++z)
                        if (static_cast<std::uint32_t>(z) == q) p[k] = inl[z];
                } else {
                    p[k] = a.rsrc[ov + q - kInlineParents];
                }
            }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) old[k] = p[k] != kNone ? pending_release(a.pending, p[k]) : 0u;
        k0 += m;
        unsigned rel = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) rel |= (old[k] == 1u ? 1u : 0u) << k;
        warp_push(wq, p, rel, nxt, next_cnt);
        if (!__any_sync(0xffffffffu, k0 < rn)) break;
    }
}

// One warp iteration over light nodes: lane `valid` holds node u.  Nodes with long
// inputs (> kHeavy entries) are only queued here -- the whole grid merges them,
// one warp per node, after the light pass of the round, so a few heavy nodes never
// serialise inside one warp.  Light nodes: inputs staged in the warp's shared
// buffer, merged per lane; junctions store P(u) -- inline when it has <= 2 input
// entries, else in pool space sized by the input length (single pass) -- and
// release their parents.  1-saddles record their merged length.  All lanes call.
__device__ __forceinline__ void count_iter(const CountArgs& a, WarpBuf wb, WarpQ& wq, PoolChunk& ch, bool valid,
                                           std::uint32_t u, std::uint32_t* nxt, unsigned long long* next_cnt,
                                           unsigned long long& done, unsigned long long* hn) {
    const int lane = threadIdx.x & 31;
    Inputs in;
    bool ovf = false;
    std::uint32_t T = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) in.len[b] = 0;
    std::uint32_t S = 0;  // staged size (lists padded to multiples of 4)
    uint4 meta = make_uint4(0u, 0u, 0u, 0u), par0 = meta, par1 = meta;
    std::uint32_t npar = 0;  // parents: their count from the rewrite's slot counters
    if (valid) {
        const uint4* nr = reinterpret_cast<const uint4*>(a.node + u);
        const uint4 d4 = a.dest[u];
        if (u < a.nj) npar = a.indeg[u];
        par0 = nr[0];
        par1 = nr[1];
        gather<true>(d4, a.rec, in, &a.flags[3]);
        T = in.len[0] + in.len[1] + in.len[2] + in.len[3];
        S = staged_size(in);
    }
    // Parents are released first: they only run next round, after the grid barrier
    // that also publishes P(u), so the release atomics overlap this node's gather and
    // merge instead of following them.  (Heavy nodes too: the heavy pass finishes them
    // within this round.)
    {
        const std::uint32_t rn = valid && u < a.nj ? npar : 0u;
        release_parents(a, wq, rn, rn > static_cast<std::uint32_t>(kInlineParents) ? a.ovoff[u] : 0ull, meta, par0,
                        par1, nxt, next_cnt);
    }
    // heavy nodes -> the round's heavy queue
    const bool heavy = valid && T > kHeavy && S + T <= wb.cap;
    {
        const unsigned hm = __ballot_sync(0xffffffffu, heavy);
        if (hm) {
            unsigned long long hb = 0;
            if (lane == 0) hb = atomicAdd(hn, static_cast<unsigned long long>(__popc(hm)));
            hb = __shfl_sync(0xffffffffu, hb, 0);
            if (heavy) a.heavy_q[hb + __popc(hm & ((1u << lane) - 1u))] = u;
        }
    }
    valid = valid && !heavy;
    const bool junction = valid && u < a.nj;
    const bool pooled = junction && T > 2;
    const std::uint64_t off = pool_alloc(a.pool, ch, pooled ? T : 0u, &a.flags[1]);
    std::uint32_t* ok = a.pool.key + (off == kBadOff ? 0 : off);
    std::uint64_t* oc = a.pool.cnt + (off == kBadOff ? 0 : off);
    JRec r;
    r.k0 = r.k1 = 0;
    r.c0 = r.c1 = 0;
    auto emit = [&](std::uint32_t o, std::uint32_t k, std::uint64_t c) {
        if (pooled) {
            if (off != kBadOff) {
                ok[o] = k;
                oc[o] = c;
            }
        } else if (o == 0) {
            r.k0 = k;
            r.c0 = c;
        } else {
            r.k1 = k;
            r.c1 = c;
        }
    };
    auto finish = [&](std::uint32_t len) {
        if (!junction) a.slen[u - a.nj] = len;
        else if (pooled) store_rec(a.rec, u, len, 1u | zword(in.z), 0u, 0u, off, 0ull);
        else store_rec(a.rec, u, len, zword(len == 0 ? __fadd_ru(in.z, 1.0f) : in.z), r.k0, r.k1, r.c0, r.c1);
    };
    // inputs larger than the warp buffer: direct merge
    if (valid && S > wb.cap) {
        const std::uint32_t len = junction ? merge<true>(in, a.pool, &ovf, emit)
                                           : merge<true>(in, a.pool, &ovf, [](std::uint32_t, std::uint32_t, std::uint64_t) {});
        finish(len);
    }
    // staged merges, in batches that fit the buffer
    unsigned todo = __ballot_sync(0xffffffffu, valid && S <= wb.cap);
    while (todo) {
        const bool mine = (todo >> lane) & 1u;
        std::uint32_t total = 0;
        const std::uint32_t base = warp_excl_scan(mine ? S : 0u, &total);
        const bool go = mine && base + S <= wb.cap;
        if (go) {
            if (junction) stage<true>(in, a.pool, wb, base);
            else stage<false>(in, a.pool, wb, base);
        }
        cp_async_wait_all();
        __syncwarp();
        if (go) {
            const std::uint32_t len =
                junction ? merge_staged<true>(in, wb, base, &ovf, emit)
                         : merge_staged<false>(in, wb, base, &ovf, [](std::uint32_t, std::uint32_t, std::uint64_t) {});
            finish(len);
        }
        __syncwarp();
        todo &= ~__ballot_sync(0xffffffffu, go);
    }
    if (junction) ++done;
    if (ovf) a.flags[0] = 1u;
}

// One heavy node, merged by the whole warp (all lanes call with the same u).
__device__ __forceinline__ void count_heavy(const CountArgs& a, WarpBuf wb, WarpQ& wq, PoolChunk& ch, std::uint32_t u,
                                            std::uint32_t* nxt, unsigned long long* next_cnt,
                                            unsigned long long& done) {
    const int lane = threadIdx.x & 31;
    const uint4* nr = reinterpret_cast<const uint4*>(a.node + u);
    const uint4 d4 = a.dest[u], meta = make_uint4(0u, 0u, 0u, 0u), par0 = nr[0], par1 = nr[1];
    Inputs h;
    gather<true>(d4, a.rec, h, &a.flags[3]);
    const std::uint32_t T = h.len[0] + h.len[1] + h.len[2] + h.len[3];
    const bool junction = u < a.nj;
    const std::uint64_t off = pool_alloc(a.pool, ch, lane == 0 && junction ? T : 0u, &a.flags[1]);
    const std::uint64_t hoff = __shfl_sync(0xffffffffu, off, 0);
    std::uint32_t at = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
        const std::uint32_t n = h.len[b];
        if (h.off[b] == kBadOff) {
            if (lane == 0 && n > 0) {
                wb.key[at] = h.k0[b];
                wb.cnt[at] = h.c0[b];
            }
            if (lane == 1 && n > 1) {
                wb.key[at + 1] = h.k1[b];
                wb.cnt[at + 1] = h.c1[b];
            }
        } else {
            for (std::uint32_t q = 4 * lane; q < n; q += 128) cp_async16(&wb.key[at + q], a.pool.key + h.off[b] + q);
            for (std::uint32_t q = 2 * lane; q < n; q += 64) cp_async16(&wb.cnt[at + q], a.pool.cnt + h.off[b] + q);
        }
        at += (n + 3u) & ~3u;
    }
    cp_async_wait_all();
    __syncwarp();
    std::uint32_t L = 0;
    bool ovf = false;
    if (!junction) L = merge_heavy(h, wb, nullptr, nullptr, &ovf);  // 1-saddle: length only
    else if (hoff != kBadOff) L = merge_heavy(h, wb, a.pool.key + hoff, a.pool.cnt + hoff, &ovf);
    if (__any_sync(0xffffffffu, ovf) && lane == 0) a.flags[0] = 1u;
    if (lane == 0) {
        if (!junction) a.slen[u - a.nj] = L;
        else store_rec(a.rec, u, L, 1u | zword(h.z), 0u, 0u, hoff, 0ull);
        if (junction) ++done;
    }
    __syncwarp();
    // (its parents were released when the light pass queued it)
}

// The round's heavy queue, one warp per node (dynamic: warps take the next node).
__device__ __forceinline__ void heavy_pass(const CountArgs& a, WarpBuf wb, WarpQ& wq, PoolChunk& ch,
                                           std::uint32_t* nxt, unsigned long long* next_cnt,
                                           unsigned long long& done, unsigned long long n, unsigned long long* head) {
    const int lane = threadIdx.x & 31;
    for (;;) {
        unsigned long long k = 0;
        if (lane == 0) k = atomicAdd(head, 1ull);
        k = __shfl_sync(0xffffffffu, k, 0);
        if (k >= n) break;
        count_heavy(a, wb, wq, ch, __ldcg(a.heavy_q + k), nxt, next_cnt, done);
    }
}

// Round 0: every node without pending children, in index order; then the frontiers.
// Two configurations of one kernel: kWide (3 blocks/SM, 384-entry
// warp buffers) runs the big early rounds, which are latency-bound and have no long
// inputs; it stops once the frontier falls below a.switch_below and leaves the state
// (round, frontier buffer, size) in a.resume.  The default configuration (2 blocks/SM,
// 1024-entry buffers for the long vectors of the tail) resumes from there.
template <bool kWide>
__global__ void __launch_bounds__(kThreads, kWide ? 3 : 2) k_count(CountArgs a) {
    extern __shared__ __align__(16) unsigned char s_dyn[];
    const WarpBuf wb = warp_buf(s_dyn, kWide ? kWarpCapWide : kWarpCap);
    __shared__ WarpQ s_q[kThreads / 32];
    __shared__ PoolChunk s_ch[kThreads / 32];
    WarpQ& wq = s_q[threadIdx.x >> 5];
    PoolChunk& ch = s_ch[threadIdx.x >> 5];
    if ((threadIdx.x & 31) == 0) {
        wq.n = 0;
        ch.base = 0;
        ch.left = 0;
    }
    __syncwarp();
    cg::grid_group grid = cg::this_grid();
    unsigned long long done = 0;
    const std::uint64_t stride = static_cast<std::uint64_t>(gridDim.x) * blockDim.x;
    const std::uint64_t wbase = (blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x) & ~31ull;
    const int lane = threadIdx.x & 31;
    std::uint32_t* cur = a.fa;
    std::uint32_t* nxt = a.fb;
    int round = 1;
    unsigned long long ncur = 0;
    // Round r's heavy queue counters are slot r % 3 (zeroed by the host, then by
    // round r - 1 for round r + 1... i.e. each round zeroes the slot of the next one).
    // A round without heavy nodes ends at its first grid barrier.
    auto finish_round = [&](int r, unsigned long long* next_cnt) {
        flush_block(s_q, nxt, next_cnt);
        grid.sync();
        const unsigned long long nh = *reinterpret_cast<volatile unsigned long long*>(&a.heavy_n[r % 3]);
        if (a.diag && grid.thread_rank() == 0 && r < kTimeline) {  // development timeline
            a.diag[7 + 3 * r] = nh;
            a.diag[8 + 3 * r] = gtimer();
        }
        if (nh) {
            heavy_pass(a, wb, wq, ch, nxt, next_cnt, done, nh, &a.heavy_head[r % 3]);
            flush_block(s_q, nxt, next_cnt);
            grid.sync();
        }
    };
    // Round 0 runs over the junctions without pending children, listed by the rewrite
    // (1-saddles: after the rounds, launch_source_len); later rounds over the frontier
    // (fb, fa, fb, ...).  One call site of the round body keeps the code compact.
    if (kWide) {
        round = 0;
        cur = const_cast<std::uint32_t*>(a.ready);
        ncur = *reinterpret_cast<const volatile unsigned long long*>(a.n_ready);
    } else {  // resume
        round = static_cast<int>(a.resume[0]);
        ncur = a.resume[1];
        if (a.resume[2]) {
            cur = a.fb;
            nxt = a.fa;
        }
    }
    while (ncur) {
        if (kWide && round > 0 && ncur < a.switch_below) break;
        unsigned long long* next_cnt = &a.cnt[(round + 1) % 3];
        if (grid.thread_rank() == 0) {
            a.cnt[(round + 2) % 3] = 0;
            a.heavy_n[(round + 1) % 3] = 0;
            a.heavy_head[(round + 1) % 3] = 0;
            if (round < kTimeline) a.stats[1 + round] = gtimer();
        }
        for (std::uint64_t base = wbase; base < ncur; base += stride) {
            const std::uint64_t f = base + lane;
            const bool valid = f < ncur;
            count_iter(a, wb, wq, ch, valid, valid ? __ldcg(cur + f) : 0u, nxt, next_cnt, done,
                       &a.heavy_n[round % 3]);
        }
        finish_round(round, next_cnt);
        if (grid.thread_rank() == 0 && a.diag && round < kTimeline) a.diag[6 + 3 * round] = ncur;
        ncur = *reinterpret_cast<volatile unsigned long long*>(next_cnt);
        ++round;
        std::uint32_t* t = cur;
        cur = nxt;
        nxt = t == a.ready ? a.fa : t;
    }
    for (int o = 16; o > 0; o >>= 1) done += __shfl_xor_sync(0xffffffffu, done, o);
    if ((threadIdx.x & 31) == 0 && done) atomicAdd(a.done, done);
    if (grid.thread_rank() == 0) {
        a.resume[0] = static_cast<unsigned long long>(round);
        a.resume[1] = ncur;
        a.resume[2] = cur == a.fb ? 1ull : 0ull;
        a.stats[0] = static_cast<unsigned long long>(round);
        if (round < kTimeline) a.stats[1 + round] = gtimer();
    }
}

// ---------------------------------------------------------------------------------
// counting, asynchronous tail: no rounds
// ---------------------------------------------------------------------------------
// Below the wide configuration's frontier threshold the rounds are latency-bound: each
// costs a node's whole dependent chain (records, pool, merge, store, release) plus grid
// barriers, ~50 us however few nodes it holds, for ~110 rounds.  The asynchronous tail
// drops the rounds: a junction is merged as soon as its last child is, by the lane that
// finished that child ("last child continues": the first parent it releases is its
// next node) or, for further released parents, by whichever warp takes them from a
// global queue.  Publication: P(u) is stored, then __threadfence(), then the parents'
// counters are decremented; a lane that takes a node (its own release, or a queue slot)
// fences before reading the children's records.  The queue is the frontier buffer the
// wide configuration stopped with: slots [0, ncur) hold its frontier, later slots are
// reserved by atomicAdd on the tail and written as node + 1 (0 = not yet written:
// zeroed at start); an idle lane claims the next slot by atomicAdd on the head and
// takes it once it is filled, while its warp goes on with the other lanes' work.
// It ends when every remaining junction is done; if none is left to take while some are
// still pending for 250 ms (a cycle: the host's count check reports it), warps give up
// (generous: a warp merging one huge vector must not look like a stall).
// Idle warps back off exponentially (64 ns .. 8 us) between polls of the counters.
struct AsyncQ {
    std::uint32_t* q;
    unsigned long long* head;
    unsigned long long* tail;
    unsigned long long* done;  // junctions finished by this kernel
    unsigned long long total;  // junctions this kernel must finish
};

// Release the parents of this lane's finished junction (P(u) already published):
// the first one that becomes ready is the lane's next node (carry), the others go to
// the queue.  All lanes call (rn = 0 for lanes without a junction).
__device__ __forceinline__ void release_async(const CountArgs& a, const AsyncQ& Q, std::uint32_t rn, std::uint64_t ov,
                                              const uint4 par0, const uint4 par1, std::uint32_t& carry) {
    const std::uint32_t inl[kInlineParents] = {par0.x, par0.y, par0.z, par0.w, par1.x, par1.y, par1.z, par1.w};
    std::uint32_t k0 = 0;
    for (;;) {
        std::uint32_t p[4], old[4];
        const std::uint32_t m = rn - k0 < 4 ? rn - k0 : 4u;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            p[k] = kNone;
            if (k < static_cast<int>(m)) {
                const std::uint32_t q = k0 + k;
                if (q < static_cast<std::uint32_t>(kInlineParents)) {
#pragma unroll
                    for (int z = 0; z < kInlineParents; ++z)
                        if (static_cast<std::uint32_t>(z) == q) p[k] = inl[z];
                } else {
                    p[k] = a.rsrc[ov + q - kInlineParents];
                }
            }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) old[k] = p[k] != kNone ? pending_release(a.pending, p[k]) : 0u;
        k0 += m;
        // the first ready parent continues on this lane; the others go to the queue,
        // all lanes' items in one reservation (the tail counter is contended)
        std::uint32_t push = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const bool ready = p[k] != kNone && old[k] == 1u;
            const bool keep = ready && carry == kNone;
            if (keep) carry = p[k];
            push |= (ready && !keep ? 1u : 0u) << k;
        }
        std::uint32_t total = 0;
        const std::uint32_t first = warp_excl_scan(static_cast<std::uint32_t>(__popc(push)), &total);
        if (total) {
            const int lane = threadIdx.x & 31;
            unsigned long long at = 0;
            if (lane == 0) at = atomicAdd(Q.tail, static_cast<unsigned long long>(total));
            at = __shfl_sync(0xffffffffu, at, 0) + first;
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if ((push >> k) & 1u) __stcg(&Q.q[at++], p[k] + 1u);  // (to the L2: the spinning reader sees it)
        }
        if (!__any_sync(0xffffffffu, k0 < rn)) break;
    }
}

// One warp iteration of the asynchronous tail: lane `valid` holds junction u.  Light
// nodes merge per lane from the warp's staging buffer, heavy ones (> kHeavy inputs)
// by the whole warp right after; then the warp publishes and releases.  All lanes call.
__device__ __forceinline__ void count_iter_async(const CountArgs& a, WarpBuf wb, WarpQ& wq, PoolChunk& ch, bool valid,
                                                 std::uint32_t u, const AsyncQ& Q, std::uint32_t& carry,
                                                 unsigned long long& done, long long* prof) {
    const int lane = threadIdx.x & 31;
    long long tp = prof ? clock64() : 0;
    auto phase = [&](int k) {  // development: cycles per phase (MSC3D_DIAG)
        if (!prof) return;
        const long long t = clock64();
        prof[k] += t - tp;
        tp = t;
    };
    Inputs in;
    bool ovf = false;
    std::uint32_t T = 0, S = 0, npar = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) in.len[b] = 0;
    uint4 par0 = make_uint4(0u, 0u, 0u, 0u), par1 = par0;
    if (valid) {
        const uint4* nr = reinterpret_cast<const uint4*>(a.node + u);
        const uint4 d4 = __ldcg(&a.dest[u]);
        npar = a.indeg[u];
        par0 = nr[0];
        par1 = nr[1];
        gather<true>(d4, a.rec, in, &a.flags[3]);
        T = in.len[0] + in.len[1] + in.len[2] + in.len[3];
        S = staged_size(in);
    }
    __syncwarp();
    phase(0);
    const bool heavy = valid && T > kHeavy && S + T <= wb.cap;
    const bool light = valid && !heavy;
    const bool pooled = light && T > 2;
    const std::uint64_t off = pool_alloc(a.pool, ch, pooled ? T : 0u, &a.flags[1]);
    __syncwarp();
    phase(1);
    std::uint32_t* ok = a.pool.key + (off == kBadOff ? 0 : off);
    std::uint64_t* oc = a.pool.cnt + (off == kBadOff ? 0 : off);
    JRec r;
    r.k0 = r.k1 = 0;
    r.c0 = r.c1 = 0;
    auto emit = [&](std::uint32_t o, std::uint32_t k, std::uint64_t c) {
        if (pooled) {
            if (off != kBadOff) {
                ok[o] = k;
                oc[o] = c;
            }
        } else if (o == 0) {
            r.k0 = k;
            r.c0 = c;
        } else {
            r.k1 = k;
            r.c1 = c;
        }
    };
    auto finish = [&](std::uint32_t len) {
        if (pooled) store_rec(a.rec, u, len, 1u | zword(in.z), 0u, 0u, off, 0ull);
        else store_rec(a.rec, u, len, zword(len == 0 ? __fadd_ru(in.z, 1.0f) : in.z), r.k0, r.k1, r.c0, r.c1);
    };
    if (light && S > wb.cap) {
        if (prof) {  // development: direct merges (inputs beyond the warp buffer) and their entries
            atomicAdd(reinterpret_cast<unsigned long long*>(Q.done) + 21, 1ull);
            atomicAdd(reinterpret_cast<unsigned long long*>(Q.done) + 22, static_cast<unsigned long long>(T));
        }
        finish(merge<true>(in, a.pool, &ovf, emit));
    }
    __syncwarp();
    unsigned todo = __ballot_sync(0xffffffffu, light && S <= wb.cap);
    while (todo) {
        const bool mine = (todo >> lane) & 1u;
        std::uint32_t total = 0;
        const std::uint32_t base = warp_excl_scan(mine ? S : 0u, &total);
        const bool go = mine && base + S <= wb.cap;
        if (go) stage<true>(in, a.pool, wb, base);
        cp_async_wait_all();
        __syncwarp();
        phase(2);
        if (go) finish(merge_staged<true>(in, wb, base, &ovf, emit));
        __syncwarp();
        phase(3);
        todo &= ~__ballot_sync(0xffffffffu, go);
        if (prof && lane == 0) atomicAdd(reinterpret_cast<unsigned long long*>(Q.done) + 23, 1ull);  // (diag: batches)
    }
    if (ovf) a.flags[0] = 1u;
    __syncwarp();
    phase(3);
    unsigned long long dummy = 0;
    for (unsigned hm = __ballot_sync(0xffffffffu, heavy); hm; hm &= hm - 1) {
        const std::uint32_t uh = __shfl_sync(0xffffffffu, u, __ffs(hm) - 1);
        count_heavy(a, wb, wq, ch, uh, nullptr, nullptr, dummy);
    }
    phase(4);
    // publish every P(u) of the warp, then release the parents
    __threadfence();
    __syncwarp();
    phase(5);
    const std::uint32_t rn = valid ? npar : 0u;
    release_async(a, Q, rn, rn > static_cast<std::uint32_t>(kInlineParents) ? a.ovoff[u] : 0ull, par0, par1, carry);
    done += static_cast<unsigned long long>(__popc(__ballot_sync(0xffffffffu, valid)));  // (warp-uniform)
    phase(6);
}

__global__ void __launch_bounds__(kThreads, 2) k_count_async(CountArgs a, unsigned long long* qctl,
                                                             const unsigned long long* n_skip,
                                                             const unsigned long long* n_predone) {
    extern __shared__ __align__(16) unsigned char s_dyn[];
    const WarpBuf wb = warp_buf(s_dyn, kWarpCap);
    __shared__ WarpQ s_q[kThreads / 32];
    __shared__ PoolChunk s_ch[kThreads / 32];
    WarpQ& wq = s_q[threadIdx.x >> 5];
    PoolChunk& ch = s_ch[threadIdx.x >> 5];
    const int lane = threadIdx.x & 31;
    if (lane == 0) {
        wq.n = 0;
        ch.base = 0;
        ch.left = 0;
    }
    __syncwarp();
    cg::grid_group grid = cg::this_grid();
    // state left by the wide configuration
    const unsigned long long ncur = a.resume[1];
    std::uint32_t* q = a.resume[2] ? a.fb : a.fa;
    const unsigned long long before = *reinterpret_cast<volatile unsigned long long*>(a.done);
    const unsigned long long total = a.nj - *n_skip - *n_predone - before;
    AsyncQ Q{q, qctl, qctl + 16, qctl + 32, total};  // (one 128-byte line each)
    for (std::uint64_t i = ncur + grid.thread_rank(); i < total; i += grid.size()) q[i] = 0u;
    for (std::uint64_t i = grid.thread_rank(); i < ncur; i += grid.size()) q[i] += 1u;  // node + 1
    if (grid.thread_rank() == 0) {
        qctl[0] = 0;
        qctl[16] = ncur;
        qctl[32] = 0;
        qctl[40] = 0;
        qctl[41] = gtimer();
        for (int k = 45; k < 64; ++k) qctl[k] = 0;
    }
    grid.sync();
    unsigned long long done = 0, flushed = 0;
    std::uint32_t carry = kNone;
    unsigned long long slot = ~0ull;  // this lane's claimed queue slot, not yet filled
    bool drained = false;             // the queue's last slot is taken: carries only
    unsigned sleep_ns = 64;  // idle back-off (thousands of idle warps must not saturate
                             // the L2 slice that holds the queue counters)
    unsigned long long last_seen = ~0ull, last_change = 0;
    long long prof_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long* prof = a.diag ? prof_acc : nullptr;
    long long t_loop = 0;
    for (;;) {
        if (prof) t_loop = clock64();
        bool has = carry != kNone;
        std::uint32_t u = carry;
        carry = kNone;
        // lanes without work and without a claim take the next slots (atomicAdd: no
        // compare-and-swap retries under contention; a slot beyond the tail is simply
        // filled later -- or never, at the end)
        const unsigned need = __ballot_sync(0xffffffffu, !has && slot == ~0ull && !drained);
        if (need) {
            unsigned long long base = 0;
            if (lane == 0) base = atomicAdd(Q.head, static_cast<unsigned long long>(__popc(need)));
            base = __shfl_sync(0xffffffffu, base, 0);
            if ((need >> lane) & 1u) {
                slot = base + __popc(need & ((1u << lane) - 1u));
                if (slot >= Q.total) {  // every node passes through at most one slot
                    slot = ~0ull;
                    drained = true;
                }
            }
        }
        if (!has && slot != ~0ull) {  // a filled slot (checked once per iteration; a volatile load:
                                      // another SM writes it meanwhile, the compiler must not keep it)
            const std::uint32_t v = *reinterpret_cast<volatile const std::uint32_t*>(&Q.q[slot]);
            if (v) {
                u = v - 1u;
                has = true;
                slot = ~0ull;
            }
        }
        if (!__any_sync(0xffffffffu, has)) {
            // nothing to do: publish this warp's count, then either all is done or wait
            if (lane == 0 && done != flushed) {
                atomicAdd(Q.done, done - flushed);
                flushed = done;
            }
            unsigned long long d = 0;
            if (lane == 0) d = *reinterpret_cast<volatile unsigned long long*>(Q.done);
            d = __shfl_sync(0xffffffffu, d, 0);
            if (d >= Q.total) break;
            const unsigned long long now = gtimer();
            if (d != last_seen) {
                last_seen = d;
                last_change = now;
            } else if (now - last_change > 250000000ull) {  // 250 ms without progress: a cycle
                if (lane == 0) atomicAdd(qctl + 40, 1ull);  // (diagnostic: warps that gave up)
                break;
            }
            __nanosleep(sleep_ns);
            sleep_ns = sleep_ns < 8192 ? 2 * sleep_ns : 8192;
            continue;
        }
        sleep_ns = 64;
        __threadfence();  // the children's records of the nodes just taken
        __syncwarp();
        if (a.diag) {  // development: warp iterations, lanes with a node, lanes from carries
            const unsigned hb = __ballot_sync(0xffffffffu, has);
            if (lane == 0) {
                atomicAdd(qctl + 45, 1ull);
                atomicAdd(qctl + 46, static_cast<unsigned long long>(__popc(hb)));
            }
        }
        if (prof) prof[7] += clock64() - t_loop;
        count_iter_async(a, wb, wq, ch, has, u, Q, carry, done, prof);
        if (lane == 0 && done - flushed >= 256) {  // (the count drives termination)
            atomicAdd(Q.done, done - flushed);
            flushed = done;
        }
    }
    if (lane == 0 && done != flushed) atomicAdd(Q.done, done - flushed);
    if (prof && lane == 0)
        for (int k = 0; k < 8; ++k) atomicAdd(qctl + 56 + k, static_cast<unsigned long long>(prof[k]));
    grid.sync();
    if (grid.thread_rank() == 0) {
        atomicAdd(a.done, *reinterpret_cast<volatile unsigned long long*>(Q.done));
        qctl[42] = gtimer();
        qctl[43] = total;
        qctl[44] = ncur;
    }
}

// The sorted (1-saddle, 2-saddle, count) output.  Light 1-saddles are merged per
// thread; heavy ones (> kHeavy input entries) are queued for k_count_write_heavy,
// one warp per 1-saddle, like the heavy junctions of k_count.
//
// kLen: the same pass computing only the merged lengths (slen) of the 1-saddles the
// walk did not finish (pending kDone) -- 1-saddles take no part in Kahn's rounds:
// nothing waits for them, so their lengths are one coalesced pass after the junctions.
constexpr int kWriteCap = 512;  // warp buffer entries of k_count_write
template <bool kLen>
__global__ void __launch_bounds__(kThreads)
k_count_write(const uint4* __restrict__ sdest, std::uint64_t n1, const JRec* __restrict__ rec,
              PoolRef pool, const std::uint64_t* __restrict__ off, std::uint32_t* __restrict__ o_one,
              std::uint32_t* __restrict__ o_two, std::uint64_t* __restrict__ o_cnt,
              std::uint32_t base_one, std::uint32_t base_two, unsigned int* __restrict__ flags,
              std::uint32_t* __restrict__ heavy_q, unsigned long long* __restrict__ heavy_n,
              const std::uint8_t* __restrict__ spending, std::uint32_t* __restrict__ slen) {
    // Light sources (<= kHeavy input entries): the warp stages its lanes' inputs in
    // shared memory (asynchronous 16-byte copies, all in flight at once) and each lane
    // merges its own from there -- instead of a chain of dependent global loads.
    // (the length pass -- few live sources, mostly short -- merges per thread from
    // global memory: measured faster than staging for it)
    if constexpr (kLen) {
        for (std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x; i < n1;
             i += static_cast<std::uint64_t>(gridDim.x) * blockDim.x) {
            if (spending[i] == kDone) continue;
            Inputs in;
            gather<false>(sdest[i], rec, in, &flags[3]);
            const std::uint32_t T = in.len[0] + in.len[1] + in.len[2] + in.len[3];
            if (T > kHeavy && staged_size(in) + T <= static_cast<std::uint32_t>(kWarpCap)) {
                heavy_q[atomicAdd(heavy_n, 1ull)] = static_cast<std::uint32_t>(i);
                continue;
            }
            bool ovf = false;
            slen[i] = merge<false>(in, pool, &ovf, [](std::uint32_t, std::uint32_t, std::uint64_t) {});
        }
        return;
    }
    extern __shared__ __align__(16) unsigned char s_dyn[];
    const WarpBuf wb = warp_buf(s_dyn, kWriteCap);
    const int lane = threadIdx.x & 31;
    const std::uint64_t stride = static_cast<std::uint64_t>(gridDim.x) * blockDim.x;
    for (std::uint64_t wbase = (blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x) & ~31ull;
         wbase < n1; wbase += stride) {
        const std::uint64_t i = wbase + lane;
        bool valid = i < n1 && !(kLen && spending[i] == kDone);
        Inputs in;
#pragma unroll
        for (int b = 0; b < 4; ++b) in.len[b] = 0;
        std::uint32_t T = 0, S = 0;
        if (valid) {
            gather<false>(sdest[i], rec, in, &flags[3]);
            T = in.len[0] + in.len[1] + in.len[2] + in.len[3];
            S = staged_size(in);
        }
        const bool heavy = valid && T > kHeavy && S + T <= static_cast<std::uint32_t>(kWarpCap);  // (heavy kernel)
        {
            const unsigned hm = __ballot_sync(0xffffffffu, heavy);
            if (hm) {
                unsigned long long hb = 0;
                if (lane == 0) hb = atomicAdd(heavy_n, static_cast<unsigned long long>(__popc(hm)));
                hb = __shfl_sync(0xffffffffu, hb, 0);
                if (heavy) heavy_q[hb + __popc(hm & ((1u << lane) - 1u))] = static_cast<std::uint32_t>(i);
            }
        }
        valid = valid && !heavy;
        bool ovf = false;
        const std::uint64_t at = (!kLen && valid) ? off[i] : 0ull;
        const std::uint32_t one = base_one + static_cast<std::uint32_t>(i);
        auto emit = [&](std::uint32_t o, std::uint32_t k, std::uint64_t c) {
            o_one[at + o] = one;
            o_two[at + o] = base_two + k;
            o_cnt[at + o] = c;
        };
        if (valid && S > wb.cap) {  // larger than the buffer (not heavy: rare): direct merge
            if (kLen) slen[i] = merge<false>(in, pool, &ovf, [](std::uint32_t, std::uint32_t, std::uint64_t) {});
            else merge<false>(in, pool, &ovf, emit);
        }
        unsigned todo = __ballot_sync(0xffffffffu, valid && S <= wb.cap);
        while (todo) {
            const bool mine = (todo >> lane) & 1u;
            std::uint32_t total = 0;
            const std::uint32_t base = warp_excl_scan(mine ? S : 0u, &total);
            const bool go = mine && base + S <= wb.cap;
            if (go) stage<!kLen>(in, pool, wb, base);
            cp_async_wait_all();
            __syncwarp();
            if (go) {
                if (kLen) slen[i] = merge_staged<false>(in, wb, base, &ovf, [](std::uint32_t, std::uint32_t, std::uint64_t) {});
                else merge_staged<true>(in, wb, base, &ovf, emit);
            }
            __syncwarp();
            todo &= ~__ballot_sync(0xffffffffu, go);
        }
        if (ovf) flags[0] = 1u;
    }
}
template <bool kLen>
__global__ void __launch_bounds__(kThreads)
k_count_write_heavy(const uint4* __restrict__ sdest, const JRec* __restrict__ rec, PoolRef pool,
                    const std::uint64_t* __restrict__ off, std::uint32_t* __restrict__ o_one,
                    std::uint32_t* __restrict__ o_two, std::uint64_t* __restrict__ o_cnt, std::uint32_t base_one,
                    std::uint32_t base_two, unsigned int* __restrict__ flags,
                    const std::uint32_t* __restrict__ heavy_q, const unsigned long long* __restrict__ heavy_n,
                    std::uint32_t* __restrict__ slen) {
    extern __shared__ __align__(16) unsigned char s_dyn[];
    const WarpBuf wb = warp_buf(s_dyn, kWarpCap);
    const int lane = threadIdx.x & 31;
    const unsigned long long n = *heavy_n;
    for (unsigned long long k = (blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x) >> 5; k < n;
         k += (static_cast<unsigned long long>(gridDim.x) * blockDim.x) >> 5) {
        const std::uint32_t i = heavy_q[k];
        Inputs h;
        gather<false>(sdest[i], rec, h, &flags[3]);
        std::uint32_t at = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const std::uint32_t m = h.len[b];
            if (h.off[b] == kBadOff) {
                if (lane == 0 && m > 0) {
                    wb.key[at] = h.k0[b];
                    wb.cnt[at] = h.c0[b];
                }
                if (lane == 1 && m > 1) {
                    wb.key[at + 1] = h.k1[b];
                    wb.cnt[at + 1] = h.c1[b];
                }
            } else {
                for (std::uint32_t q = 4 * lane; q < m; q += 128) cp_async16(&wb.key[at + q], pool.key + h.off[b] + q);
                for (std::uint32_t q = 2 * lane; q < m; q += 64) cp_async16(&wb.cnt[at + q], pool.cnt + h.off[b] + q);
            }
            at += (m + 3u) & ~3u;
        }
        cp_async_wait_all();
        __syncwarp();
        bool ovf = false;
        if (kLen) {
            const std::uint32_t L = merge_heavy(h, wb, nullptr, nullptr, &ovf);
            if (lane == 0) slen[i] = L;
            __syncwarp();
            continue;
        }
        const std::uint64_t o = off[i];
        const std::uint32_t L = merge_heavy(h, wb, o_two + o, o_cnt + o, &ovf);
        for (std::uint32_t t = lane; t < L; t += 32) {
            o_one[o + t] = base_one + i;
            o_two[o + t] += base_two;
        }
        if (__any_sync(0xffffffffu, ovf) && lane == 0) flags[0] = 1u;
        __syncwarp();
    }
}

}  // namespace

// ---------------------------------------------------------------------------------
// host wrappers
// ---------------------------------------------------------------------------------
namespace {
EGrid egrid(const Dims& d) {
    return EGrid{static_cast<std::uint32_t>(d.nx), static_cast<std::uint32_t>(d.nx * d.ny)};
}
}  // namespace

int launch_succ_table(const std::uint8_t* codes, const Dims& d, std::uint16_t* succ, cudaStream_t s, int num_sms) {
    const std::uint64_t rows = static_cast<std::uint64_t>(d.ny) * d.nz;
    if (rows == 0) return MSC3D_OK;
    // persistent blocks walking the rows in order (the resident blocks work on a
    // compact window of rows: neighbouring rows share their code lines in L2)
    static std::uint8_t* lut[64] = {nullptr};
    int dev = 0;
    MSC3D_CUDA_TRY(cudaGetDevice(&dev));
    if (dev < 0 || dev >= 64) return MSC3D_ERR_INVALID;
    if (!lut[dev]) {
        MSC3D_CUDA_TRY(cudaMalloc(&lut[dev], 12 * 256));
        k_succ_lut<<<12, 256, 0, s>>>(lut[dev]);
        count_launch();
    }
    const unsigned grid = static_cast<unsigned>(std::min<std::uint64_t>(rows, static_cast<std::uint64_t>(num_sms) * 8));
    k_succ_table<<<grid, 256, 0, s>>>(codes, d, reinterpret_cast<const uint4*>(lut[dev]), succ);
    count_launch();
    MSC3D_CUDA_TRY(cudaGetLastError());
    return MSC3D_OK;
}

int coop_blocks(const void* fn, int num_sms, int* grid, std::size_t smem = 0) {
    int per_sm = 0;
    MSC3D_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kThreads, smem));
    if (per_sm <= 0) return MSC3D_ERR_CUDA;
    *grid = per_sm * num_sms;
    return MSC3D_OK;
}

int launch_reach(const std::uint16_t* succ, const Dims& d, unsigned int* bitmap, std::uint32_t* fa,
                 std::uint32_t* fb, unsigned long long cap, unsigned long long* cnt, unsigned long long* stats,
                 cudaStream_t s, int num_sms) {
    int grid = 0;
    const int rc = coop_blocks(reinterpret_cast<const void*>(k_reach), num_sms, &grid);
    if (rc != MSC3D_OK) return rc;
    EGrid g = egrid(d);
    void* args[] = {&succ, &g, &bitmap, &fa, &fb, &cnt, &stats, &cap};
    MSC3D_CUDA_TRY(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k_reach), dim3(grid), dim3(kThreads),
                                               args, 0, s));
    count_launch();
    return MSC3D_OK;
}

int launch_junction_bits(const std::uint16_t* succ, const unsigned int* bitmap, std::uint64_t nwords,
                         unsigned int* jbits, std::uint32_t* jcnt, unsigned long long* nodes, cudaStream_t s,
                         int num_sms) {
    if (nwords == 0) return MSC3D_OK;
    k_junction_bits<<<grid_for(nwords, num_sms, 16), kThreads, 0, s>>>(succ, bitmap, nwords, jbits, jcnt, nodes);
    count_launch();
    MSC3D_CUDA_TRY(cudaGetLastError());
    return MSC3D_OK;
}

int launch_junction_list(const unsigned int* jbits, std::uint64_t nwords, const std::uint64_t* woff, void* jrank,
                         std::uint32_t* jlist, cudaStream_t s, int num_sms) {
    if (nwords == 0) return MSC3D_OK;
    k_junction_list<<<grid_for(nwords, num_sms, 16), kThreads, 0, s>>>(jbits, nwords, woff, jlist, static_cast<uint2*>(jrank));
    count_launch();
    MSC3D_CUDA_TRY(cudaGetLastError());
    return MSC3D_OK;
}

int launch_walk(const std::uint16_t* succ, const Dims& d, const void* jrank,
                const std::uint32_t* tmap, const void* trank, const std::uint32_t* jlist, const void* srcs, int id_width,
                std::uint64_t n, void* node, std::uint8_t* pending, unsigned int* flags, void* rec,
                std::uint32_t* slen, unsigned int* predone, unsigned long long* n_predone, std::uint32_t* fwd,
                unsigned int* ptbits, cudaStream_t s, int num_sms) {
    if (n == 0) return MSC3D_OK;
    WalkCtx c{succ, egrid(d), static_cast<const uint2*>(jrank), tmap, static_cast<const uint2*>(trank), d.n_cells,
              d.fnx, d.fny, static_cast<std::uint32_t>(d.nx), static_cast<std::uint32_t>(d.ny), static_cast<std::uint64_t>(d.ex),
              static_cast<std::uint64_t>(d.exy)};
    auto* nr = static_cast<uint4*>(node);  // the nodes' destination records
    auto* r4 = static_cast<uint4*>(rec);
    if (id_width == 4)
        k_walk<std::uint32_t><<<static_cast<unsigned>((n + 127) / 128), 128, 0, s>>>(
            c, d, jlist, static_cast<const std::uint32_t*>(srcs), n, nr, pending, flags, r4, slen, predone, n_predone, fwd, ptbits);
    else
        k_walk<std::uint64_t><<<static_cast<unsigned>((n + 127) / 128), 128, 0, s>>>(
            c, d, jlist, static_cast<const std::uint64_t*>(srcs), n, nr, pending, flags, r4, slen, predone, n_predone, fwd, ptbits);
    count_launch();
    MSC3D_CUDA_TRY(cudaGetLastError());
    return MSC3D_OK;
}

int launch_term_rank(const void* list, std::uint64_t n, int id_width, std::uint64_t n_cells, void* trank,
                     cudaStream_t s, int num_sms) {
    MSC3D_CUDA_TRY(cudaMemsetAsync(trank, 0, (n_cells / 32 + 1) * 8, s));
    if (n == 0) return MSC3D_OK;
    auto* tr = static_cast<uint2*>(trank);
    if (id_width == 4)
        k_term_rank<<<grid_for(n, num_sms), kThreads, 0, s>>>(static_cast<const std::uint32_t*>(list), n, tr);
    else
        k_term_rank<<<grid_for(n, num_sms), kThreads, 0, s>>>(static_cast<const std::uint64_t*>(list), n, tr);
    count_launch();
    MSC3D_CUDA_TRY(cudaGetLastError());
    return MSC3D_OK;
}

int node_rec_bytes() { return static_cast<int>(sizeof(NodeRec)); }


int launch_rewrite(void* node, void* dest, std::uint64_t nj, std::uint64_t n_nodes, const std::uint32_t* fwd,
                   const unsigned int* ptbits, const unsigned int* predone, std::uint8_t* pending, std::uint32_t* indeg, void* ovq, unsigned long long* ovq_n,
                   std::uint64_t ovq_cap, unsigned long long* n_skip, std::uint32_t* ready,
                   unsigned long long* n_ready, cudaStream_t s, int num_sms) {
    if (n_nodes == 0) return MSC3D_OK;
    k_rewrite<<<grid_full((n_nodes + kRwPer - 1) / kRwPer), kThreads, 0, s>>>(static_cast<NodeRec*>(node), static_cast<uint4*>(dest), nj, n_nodes, fwd, ptbits, predone,
                                                      pending, indeg, static_cast<uint4*>(ovq), ovq_n, ovq_cap, n_skip,
                                                      ready, n_ready);
    count_launch();
    MSC3D_CUDA_TRY(cudaGetLastError());
    return MSC3D_OK;
}

int launch_parent_overflow(const std::uint32_t* indeg, std::uint64_t nj, std::uint64_t* ovoff,
                           unsigned long long* total, cudaStream_t s, int num_sms) {
    MSC3D_CUDA_TRY(cudaMemsetAsync(total, 0, 8, s));
    if (nj == 0) return MSC3D_OK;
    k_parent_overflow<<<grid_for(nj, num_sms), kThreads, 0, s>>>(indeg, nj, ovoff, total);
    count_launch();
    MSC3D_CUDA_TRY(cudaGetLastError());
    return MSC3D_OK;
}

int launch_fill_parents(void* node, std::uint64_t nj, const std::uint32_t* indeg, const std::uint64_t* ovoff,
                        const void* ovq, std::uint64_t n_ovq, std::uint32_t* rsrc, cudaStream_t s, int num_sms) {
    auto* nr = static_cast<NodeRec*>(node);
    (void)nr;
    (void)nj;
    (void)indeg;  // parent counts are read from the rewrite's slot counters directly
    if (n_ovq) {
        k_fill_overflow<<<grid_for(n_ovq, num_sms), kThreads, 0, s>>>(static_cast<const uint4*>(ovq), n_ovq, ovoff,
                                                                       rsrc);
        count_launch();
    }
    MSC3D_CUDA_TRY(cudaGetLastError());
    return MSC3D_OK;
}

int count_rec_bytes() { return static_cast<int>(sizeof(JRec)); }
int count_arenas() { return kArenas; }

int launch_count(const CountLaunch& L, cudaStream_t s, int num_sms) {
    CountArgs a;
    a.node = static_cast<const NodeRec*>(L.node);
    a.pending = L.pending;
    a.pending0 = L.pending0;
    a.rsrc = L.rsrc;
    a.rec = static_cast<JRec*>(L.rec);
    a.pool = PoolRef{L.pool_key, L.pool_cnt, L.pool_top, L.arena_cap};
    a.slen = L.slen;
    a.nj = L.nj;
    a.n1 = L.n1;
    a.fa = L.fa;
    a.fb = L.fb;
    a.cnt = L.cnt;
    a.stats = L.stats;
    a.done = L.done;
    a.flags = L.flags;
    a.diag = L.diag;
    a.heavy_q = L.heavy_q;
    a.dest = static_cast<const uint4*>(L.dest);
    a.ready = L.ready;
    a.n_ready = L.n_ready;
    a.heavy_n = L.heavy_rounds;
    a.heavy_head = L.heavy_rounds + 3;
    if (L.nj + L.n1 == 0) return MSC3D_OK;
    a.switch_below = L.switch_below;
    a.indeg = L.indeg;
    a.ovoff = L.ovoff;
    a.resume = L.resume;
    // early rounds: the wide configuration; then the default one resumes
    const std::size_t smem_w = warp_buf_bytes(kWarpCapWide) * (kThreads / 32);
    const std::size_t smem_d = warp_buf_bytes(kWarpCap) * (kThreads / 32);
    const void* kw = reinterpret_cast<const void*>(k_count<true>);
    const void* kd = reinterpret_cast<const void*>(k_count<false>);
    MSC3D_CUDA_TRY(cudaFuncSetAttribute(kw, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_w)));
    MSC3D_CUDA_TRY(cudaFuncSetAttribute(kd, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_d)));
    int grid = 0;
    int rc = coop_blocks(kw, num_sms, &grid, smem_w);
    if (rc != MSC3D_OK) return rc;
    void* args[] = {&a};
    MSC3D_CUDA_TRY(cudaLaunchCooperativeKernel(kw, dim3(grid), dim3(kThreads), args, smem_w, s));
    if (L.async_tail) {  // the tail without rounds
        const void* ka = reinterpret_cast<const void*>(k_count_async);
        MSC3D_CUDA_TRY(cudaFuncSetAttribute(ka, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_d)));
        rc = coop_blocks(ka, num_sms, &grid, smem_d);
        if (rc != MSC3D_OK) return rc;
        unsigned long long* qctl = L.qctl;
        const unsigned long long* nsk = L.n_skip;
        const unsigned long long* npd = L.n_predone;
        void* aargs[] = {&a, &qctl, &nsk, &npd};
        MSC3D_CUDA_TRY(cudaLaunchCooperativeKernel(ka, dim3(grid), dim3(kThreads), aargs, smem_d, s));
        count_launch(2);
        return MSC3D_OK;
    }
    rc = coop_blocks(kd, num_sms, &grid, smem_d);
    if (rc != MSC3D_OK) return rc;
    MSC3D_CUDA_TRY(cudaLaunchCooperativeKernel(kd, dim3(grid), dim3(kThreads), args, smem_d, s));
    count_launch(2);
    return MSC3D_OK;
}

namespace {
template <bool kLen>
int count_write_impl(const CountLaunch& L, const std::uint64_t* off, std::uint32_t* o_one, std::uint32_t* o_two,
                     std::uint64_t* o_cnt, std::uint32_t base_one, std::uint32_t base_two, cudaStream_t s,
                     int num_sms) {
    if (L.n1 == 0) return MSC3D_OK;
    const uint4* snode = static_cast<const uint4*>(L.dest) + L.nj;
    const PoolRef pool{L.pool_key, L.pool_cnt, L.pool_top, L.arena_cap};
    MSC3D_CUDA_TRY(cudaMemsetAsync(L.heavy_n, 0, 8, s));
    const std::size_t smem_l = kLen ? 0 : warp_buf_bytes(kWriteCap) * (kThreads / 32);
    MSC3D_CUDA_TRY(cudaFuncSetAttribute(reinterpret_cast<const void*>(k_count_write<kLen>),
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_l)));
    k_count_write<kLen><<<grid_full(L.n1), kThreads, smem_l, s>>>(snode, L.n1, static_cast<const JRec*>(L.rec), pool,
                                                                  off, o_one, o_two, o_cnt, base_one, base_two, L.flags,
                                                                  L.heavy_q, L.heavy_n, L.pending0 + L.nj, L.slen);
    const std::size_t smem = warp_buf_bytes(kWarpCap) * (kThreads / 32);
    MSC3D_CUDA_TRY(cudaFuncSetAttribute(reinterpret_cast<const void*>(k_count_write_heavy<kLen>),
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    k_count_write_heavy<kLen><<<num_sms * 2, kThreads, smem, s>>>(snode, static_cast<const JRec*>(L.rec), pool, off,
                                                                  o_one, o_two, o_cnt, base_one, base_two, L.flags,
                                                                  L.heavy_q, L.heavy_n, L.slen);
    count_launch(2);
    MSC3D_CUDA_TRY(cudaGetLastError());
    return MSC3D_OK;
}
}  // namespace

int launch_source_len(const CountLaunch& L, cudaStream_t s, int num_sms) {
    return count_write_impl<true>(L, nullptr, nullptr, nullptr, nullptr, 0, 0, s, num_sms);
}

int launch_count_write(const CountLaunch& L, const std::uint64_t* off, std::uint32_t* o_one, std::uint32_t* o_two,
                       std::uint64_t* o_cnt, std::uint32_t base_one, std::uint32_t base_two, cudaStream_t s,
                       int num_sms) {
    return count_write_impl<false>(L, off, o_one, o_two, o_cnt, base_one, base_two, s, num_sms);
}

}  // namespace msc3d_dev

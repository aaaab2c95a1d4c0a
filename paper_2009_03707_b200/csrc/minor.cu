// Stage-level saddle APIs on the device:
//   * build_minor (saddle_graph.cpp:121-217): junction list in cell order, one walk
//     per 1-saddle / junction branch, parallel branches merged into multiplicities;
//   * count_paths on an explicit DagMinor (path_matrix.cpp:188-219) and
//     sp_multiply / sp_add (path_matrix.cpp:115-186): one generic "merge rows"
//     engine -- every output row is the sum of scaled input rows (a terminal
//     contributes a single (key, mult) entry): expand -> segmented sort -> reduce,
//     exact u64 with sticky overflow.
// The whole-field pipeline (compute) does not use this engine; it runs the branch
// walks and the Kahn counting kernels of dag.cu.
#include <algorithm>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "common.cuh"
#include "ctx.cuh"
#include "kernels.cuh"
#include "stages.cuh"

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

// jlist_de[k] = dense edge of junction cell k; jidx[dense edge] = k
template <typename IdT>
__global__ void k_junction_dense(const IdT* __restrict__ cells, std::uint64_t n, Dims d,
                                 std::uint32_t* __restrict__ jlist, std::uint32_t* __restrict__ jidx) {
    GRID_STRIDE(k, n) {
        const Coord c = unpack(d, cells[k]);
        const int axis = (c.x & 1) ? 0 : ((c.y & 1) ? 1 : 2);
        const std::uint32_t de =
            3u * static_cast<std::uint32_t>((c.x >> 1) + d.nx * ((c.y >> 1) + d.ny * (c.z >> 1))) + axis;
        jlist[k] = de;
        jidx[de] = static_cast<std::uint32_t>(k);
    }
}

// Per origin: its (<= 4) branch destinations sorted, equal ones merged.  Pass 1
// counts junction / 2-saddle destinations, pass 2 writes (src, dst, mult) rows.
__device__ __forceinline__ int origin_runs(const std::uint32_t* __restrict__ dest, std::uint64_t i,
                                           std::uint32_t v[4], std::uint32_t m[4]) {
    const uint4 d4 = reinterpret_cast<const uint4*>(dest)[i];
    std::uint32_t a[4] = {d4.x, d4.y, d4.z, d4.w};
    // sort 4 (kNone sorts last; junctions (bit 31 clear) before 2-saddles)
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int q = 0; q < 3 - p; ++q) {
            const std::uint32_t lo = min(a[q], a[q + 1]), hi = max(a[q], a[q + 1]);
            a[q] = lo;
            a[q + 1] = hi;
        }
    int n = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        if (a[k] == kNone) continue;
        if (n > 0 && v[n - 1] == a[k]) {
            ++m[n - 1];
        } else {
            v[n] = a[k];
            m[n] = 1;
            ++n;
        }
    }
    return n;
}

__global__ void k_minor_count(const std::uint32_t* __restrict__ dest, std::uint64_t n,
                              std::uint32_t* __restrict__ cnt_j, std::uint32_t* __restrict__ cnt_t) {
    GRID_STRIDE(i, n) {
        std::uint32_t v[4], m[4];
        const int r = origin_runs(dest, i, v, m);
        std::uint32_t nj = 0, nt = 0;
        for (int k = 0; k < r; ++k) {
            if (v[k] & kTerm) ++nt;
            else ++nj;
        }
        cnt_j[i] = nj;
        cnt_t[i] = nt;
    }
}

__global__ void k_minor_write(const std::uint32_t* __restrict__ dest, std::uint64_t n,
                              const std::uint64_t* __restrict__ off_j, const std::uint64_t* __restrict__ off_t,
                              std::uint32_t* __restrict__ js, std::uint32_t* __restrict__ jd,
                              std::uint64_t* __restrict__ jm, std::uint32_t* __restrict__ ts,
                              std::uint32_t* __restrict__ td, std::uint64_t* __restrict__ tm) {
    GRID_STRIDE(i, n) {
        std::uint32_t v[4], m[4];
        const int r = origin_runs(dest, i, v, m);
        std::uint64_t aj = off_j[i], at = off_t[i];
        for (int k = 0; k < r; ++k) {
            if (v[k] & kTerm) {
                ts[at] = static_cast<std::uint32_t>(i);
                td[at] = v[k] & ~kTerm;
                tm[at] = m[k];
                ++at;
            } else {
                js[aj] = static_cast<std::uint32_t>(i);
                jd[aj] = v[k];
                jm[aj] = m[k];
                ++aj;
            }
        }
    }
}

// ---- the generic merge-rows engine ---------------------------------------------------
// A reference into the key/count pool: len entries at off scaled by mult, or (when
// len == kOne) the single entry (key, 1) scaled by mult.
constexpr std::uint32_t kOne = 0xffffffffu;
struct Ref {
    std::uint64_t off;
    std::uint64_t mult;
    std::uint32_t len;
    std::uint32_t key;
};

__device__ __forceinline__ std::uint64_t ref_len(const Ref& r) { return r.len == kOne ? 1ull : r.len; }

__global__ void k_expand_count(std::uint64_t rows, const std::uint64_t* __restrict__ roff,
                               const Ref* __restrict__ refs, std::uint32_t* __restrict__ cnt) {
    GRID_STRIDE(r, rows) {
        std::uint64_t n = 0;
        for (std::uint64_t k = roff[r]; k < roff[r + 1]; ++k) n += ref_len(refs[k]);
        cnt[r] = static_cast<std::uint32_t>(n);
    }
}

__global__ void k_expand(std::uint64_t rows, const std::uint64_t* __restrict__ roff, const Ref* __restrict__ refs,
                         const std::uint32_t* __restrict__ pkey, const std::uint64_t* __restrict__ pcnt,
                         const std::uint64_t* __restrict__ eoff, std::uint64_t* __restrict__ ekey,
                         std::uint64_t* __restrict__ eval, unsigned int* __restrict__ flags) {
    GRID_STRIDE(r, rows) {
        std::uint64_t at = eoff[r];
        const std::uint64_t base = at;
        for (std::uint64_t k = roff[r]; k < roff[r + 1]; ++k) {
            const Ref f = refs[k];
            const std::uint64_t n = ref_len(f);
            for (std::uint64_t j = 0; j < n; ++j) {
                const std::uint32_t key = f.len == kOne ? f.key : pkey[f.off + j];
                const std::uint64_t c = f.len == kOne ? 1ull : pcnt[f.off + j];
                const std::uint64_t v = c * f.mult;
                if (__umul64hi(c, f.mult) != 0) flags[0] = 1u;
                ekey[at] = (static_cast<std::uint64_t>(key) << 32) | (at - base);
                eval[at] = v;
                ++at;
            }
        }
    }
}

// pass 0: count distinct keys with a non-zero sum; pass 1: write them
template <bool kWrite>
__global__ void k_reduce(std::uint64_t rows, const std::uint64_t* __restrict__ eoff, std::uint64_t etotal,
                         const std::uint64_t* __restrict__ ekey, const std::uint64_t* __restrict__ eval,
                         std::uint32_t* __restrict__ ocnt, const std::uint64_t* __restrict__ ooff,
                         std::uint32_t* __restrict__ okey, std::uint64_t* __restrict__ oval,
                         unsigned int* __restrict__ flags) {
    GRID_STRIDE(r, rows) {
        const std::uint64_t b = eoff[r], e = r + 1 < rows ? eoff[r + 1] : etotal;
        std::uint64_t at = kWrite ? ooff[r] : 0;
        std::uint32_t n = 0;
        for (std::uint64_t i = b; i < e;) {
            const std::uint32_t key = static_cast<std::uint32_t>(ekey[i] >> 32);
            std::uint64_t sum = 0;
            bool ovf = false;
            for (; i < e && static_cast<std::uint32_t>(ekey[i] >> 32) == key; ++i) {
                const std::uint64_t v = eval[b + static_cast<std::uint32_t>(ekey[i])];
                const std::uint64_t s2 = sum + v;
                ovf |= s2 < sum;
                sum = s2;
            }
            if (ovf) flags[0] = 1u;
            if (sum == 0) continue;
            if (kWrite) {
                okey[at] = key;
                oval[at] = sum;
                ++at;
            }
            ++n;
        }
        if (!kWrite) ocnt[r] = n;
    }
}

// Refs of the level's junction rows (count_minor): dests in CSR (dst | kTerm for
// 2-saddles, junction index otherwise) with multiplicities; junction children's
// vectors are (P_off, P_len) in the pool.
__global__ void k_level_refs(const std::uint32_t* __restrict__ rows, std::uint64_t nrows,
                             const std::uint64_t* __restrict__ csr_off, const std::uint32_t* __restrict__ csr_dst,
                             const std::uint64_t* __restrict__ csr_mult, const std::uint64_t* __restrict__ roff,
                             const std::uint64_t* __restrict__ P_off, const std::uint32_t* __restrict__ P_len,
                             Ref* __restrict__ refs) {
    GRID_STRIDE(i, nrows) {
        const std::uint32_t o = rows[i];
        std::uint64_t at = roff[i];
        for (std::uint64_t k = csr_off[o]; k < csr_off[o + 1]; ++k) {
            const std::uint32_t t = csr_dst[k];
            Ref f;
            f.mult = csr_mult[k];
            if (t & kTerm) {
                f.len = kOne;
                f.key = t & ~kTerm;
                f.off = 0;
            } else {
                f.len = P_len[t];
                f.key = 0;
                f.off = P_off[t];
            }
            refs[at++] = f;
        }
    }
}

__global__ void k_set_rows_P(const std::uint32_t* __restrict__ rows, std::uint64_t nrows, std::uint64_t base,
                             const std::uint64_t* __restrict__ ooff, const std::uint32_t* __restrict__ ocnt,
                             std::uint64_t* __restrict__ P_off, std::uint32_t* __restrict__ P_len) {
    GRID_STRIDE(i, nrows) {
        P_off[rows[i]] = base + ooff[i];
        P_len[rows[i]] = ocnt[i];
    }
}

// Forward saturating path totals into junctions (A* row sums): F(j) = sum over
// predecessors; saturates at 2^64 (flag) -> exact per-source check needed.
__global__ void k_forward_level(const std::uint32_t* __restrict__ rows, std::uint64_t nrows,
                                const std::uint64_t* __restrict__ pred_off, const std::uint32_t* __restrict__ pred_src,
                                const std::uint64_t* __restrict__ pred_mult, std::uint64_t* __restrict__ F,
                                unsigned int* __restrict__ sat) {
    GRID_STRIDE(i, nrows) {
        const std::uint32_t j = rows[i];
        std::uint64_t s = F[j];  // pre-seeded with the 1-saddle -> j multiplicities
        bool o = s == ~0ull;
        for (std::uint64_t k = pred_off[j]; k < pred_off[j + 1]; ++k) {
            const std::uint64_t f = F[pred_src[k]];
            const std::uint64_t p = f * pred_mult[k];
            if (f == ~0ull || __umul64hi(f, pred_mult[k]) != 0) o = true;
            const std::uint64_t s2 = s + p;
            if (s2 < s) o = true;
            s = s2;
        }
        F[j] = o ? ~0ull : s;
        if (o) *sat = 1u;
    }
}

// Exact A* overflow check, one thread per 1-saddle of rows [row0, row0 + n1) (a batch:
// A holds n1 dense rows of nj counts), junctions in topological order.
__global__ void k_forward_exact(std::uint64_t row0, std::uint64_t n1, std::uint64_t nj, const std::uint32_t* __restrict__ topo,
                                std::uint64_t ntopo, const std::uint64_t* __restrict__ pred_off,
                                const std::uint32_t* __restrict__ pred_src, const std::uint64_t* __restrict__ pred_mult,
                                const std::uint64_t* __restrict__ s_off, const std::uint32_t* __restrict__ s_dst,
                                const std::uint64_t* __restrict__ s_mult, std::uint64_t* __restrict__ A,
                                unsigned int* __restrict__ flags) {
    GRID_STRIDE(r, n1) {
        const std::uint64_t i = row0 + r;
        std::uint64_t* a = A + r * nj;
        for (std::uint64_t j = 0; j < nj; ++j) a[j] = 0;
        for (std::uint64_t k = s_off[i]; k < s_off[i + 1]; ++k) {
            const std::uint32_t t = s_dst[k];
            if (t & kTerm) continue;
            const std::uint64_t s2 = a[t] + s_mult[k];
            if (s2 < a[t]) flags[0] = 1u;
            a[t] = s2;
        }
        for (std::uint64_t q = 0; q < ntopo; ++q) {
            const std::uint32_t j = topo[q];
            std::uint64_t s = a[j];
            for (std::uint64_t k = pred_off[j]; k < pred_off[j + 1]; ++k) {
                const std::uint64_t f = a[pred_src[k]];
                if (__umul64hi(f, pred_mult[k]) != 0) flags[0] = 1u;
                const std::uint64_t s2 = s + f * pred_mult[k];
                if (s2 < s) flags[0] = 1u;
                s = s2;
            }
            a[j] = s;
        }
    }
}

__global__ void k_sp_refs(int op, std::uint64_t rows, const std::uint64_t* __restrict__ xp,
                          const std::uint32_t* __restrict__ xc, const std::uint64_t* __restrict__ xv,
                          const std::uint64_t* __restrict__ yp, std::uint64_t ybase, const std::uint64_t* __restrict__ roff,
                          Ref* __restrict__ refs) {
    GRID_STRIDE(r, rows) {
        std::uint64_t at = roff[r];
        if (op == 0) {  // row r of x*y: sum over x[r, k] * y[k, :]
            for (std::uint64_t p = xp[r]; p < xp[r + 1]; ++p) {
                const std::uint32_t k = xc[p];
                Ref f;
                f.off = ybase + yp[k];
                f.len = static_cast<std::uint32_t>(yp[k + 1] - yp[k]);
                f.mult = xv[p];
                f.key = 0;
                refs[at++] = f;
            }
        } else {  // row r of x+y
            Ref f;
            f.off = xp[r];
            f.len = static_cast<std::uint32_t>(xp[r + 1] - xp[r]);
            f.mult = 1;
            f.key = 0;
            refs[at++] = f;
            f.off = ybase + yp[r];
            f.len = static_cast<std::uint32_t>(yp[r + 1] - yp[r]);
            refs[at++] = f;
        }
    }
}

}  // namespace

}  // namespace msc3d_dev

// =====================================================================================
// stage functions
// =====================================================================================
namespace msc3d_stage {

using msc3d_dev::Dims;
using msc3d_dev::Ref;

#define TRY(x)                              \
    do {                                    \
        const int _rc = (x);                \
        if (_rc != MSC3D_OK) return _rc;    \
    } while (0)

namespace {

template <typename T>
int upload(msc3d_ctx* ctx, const std::string& name, const std::vector<T>& v) {
    void* p = ctx->ensure(name, v.size(), sizeof(T));
    if (!p) return MSC3D_ERR_NOMEM;
    if (!v.empty()) MSC3D_CUDA_TRY(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, ctx->stream));
    return MSC3D_OK;
}

// Merge `rows` output rows whose refs (CSR roff over refs) point into the pool
// (pkey/pcnt).  Result rows land in out_key/out_cnt ("<prefix>.key/.cnt") with per-row
// offsets "<prefix>.off" and lengths "<prefix>.len"; *out_total = entries written.
int merge_rows(msc3d_ctx* ctx, std::uint64_t rows, const std::uint64_t* roff, const Ref* refs,
               const std::uint32_t* pkey, const std::uint64_t* pcnt, const std::string& prefix,
               std::uint64_t* out_total) {
    const cudaStream_t s = ctx->stream;
    const int sms = ctx->num_sms;
    *out_total = 0;
    auto* ecnt = static_cast<std::uint32_t*>(ctx->ensure(prefix + ".ecnt", rows, 4));
    auto* eoff = static_cast<std::uint64_t*>(ctx->ensure(prefix + ".eoff", rows, 8));
    auto* ocnt = static_cast<std::uint32_t*>(ctx->ensure(prefix + ".len", rows, 4));
    auto* ooff = static_cast<std::uint64_t*>(ctx->ensure(prefix + ".off", rows, 8));
    if (!ecnt || !eoff || !ocnt || !ooff) return MSC3D_ERR_NOMEM;
    if (rows == 0) return MSC3D_OK;
    auto* flags = reinterpret_cast<unsigned int*>(ctx->d_small + 26);
    msc3d_dev::k_expand_count<<<msc3d_dev::grid_for(rows, sms), msc3d_dev::kThreads, 0, s>>>(rows, roff, refs, ecnt);
    msc3d_dev::count_launch();
    TRY(msc3d_dev::scan_u32(ecnt, rows, eoff, ctx->d_small, ctx->ws, s));
    TRY(ctx->fetch_small(1));
    const std::uint64_t E = ctx->h_small[0];
    auto* ekey = static_cast<std::uint64_t*>(ctx->ensure(prefix + ".ekey", E, 8));
    auto* eval = static_cast<std::uint64_t*>(ctx->ensure(prefix + ".eval", E, 8));
    auto* scratch = static_cast<std::uint64_t*>(ctx->ensure(prefix + ".scratch", E, 8));
    auto* large = static_cast<std::uint32_t*>(ctx->ensure(prefix + ".large", rows, 4));
    if (!ekey || !eval || !scratch || !large) return MSC3D_ERR_NOMEM;
    msc3d_dev::k_expand<<<msc3d_dev::grid_for(rows, sms), msc3d_dev::kThreads, 0, s>>>(rows, roff, refs, pkey, pcnt,
                                                                                      eoff, ekey, eval, flags);
    msc3d_dev::count_launch();
    TRY(msc3d_dev::launch_bucket_sort(eoff, rows, E, ekey, scratch, large,
                                      reinterpret_cast<unsigned long long*>(ctx->d_small + 35), ctx->h_small + 35,
                                      s, sms));
    msc3d_dev::k_reduce<false><<<msc3d_dev::grid_for(rows, sms), msc3d_dev::kThreads, 0, s>>>(
        rows, eoff, E, ekey, eval, ocnt, nullptr, nullptr, nullptr, flags);
    msc3d_dev::count_launch();
    TRY(msc3d_dev::scan_u32(ocnt, rows, ooff, ctx->d_small, ctx->ws, s));
    TRY(ctx->fetch_small(1));
    const std::uint64_t O = ctx->h_small[0];
    auto* okey = static_cast<std::uint32_t*>(ctx->ensure(prefix + ".key", O, 4));
    auto* oval = static_cast<std::uint64_t*>(ctx->ensure(prefix + ".cnt", O, 8));
    if (!okey || !oval) return MSC3D_ERR_NOMEM;
    msc3d_dev::k_reduce<true><<<msc3d_dev::grid_for(rows, sms), msc3d_dev::kThreads, 0, s>>>(
        rows, eoff, E, ekey, eval, nullptr, ooff, okey, oval, flags);
    msc3d_dev::count_launch();
    MSC3D_CUDA_TRY(cudaGetLastError());
    *out_total = O;
    return MSC3D_OK;
}

}  // namespace

int load_marked(msc3d_ctx* ctx, const std::uint8_t* host_marked, const void* ones, std::uint64_t n1,
                const void* twos, std::uint64_t n2) {
    if (!ctx->have_dims || !ctx->find("codes")) return MSC3D_ERR_STATE;
    const Dims& d = ctx->dims;
    const int w = ctx->id_width();
    void* m = ctx->ensure("marked", d.n_cells, 1);
    void* a = ctx->ensure("one_saddles", n1, w);
    void* b = ctx->ensure("two_saddles", n2, w);
    if (!m || !a || !b) return MSC3D_ERR_NOMEM;
    MSC3D_CUDA_TRY(cudaMemcpyAsync(m, host_marked, d.n_cells, cudaMemcpyHostToDevice, ctx->stream));
    if (n1) MSC3D_CUDA_TRY(cudaMemcpyAsync(a, ones, n1 * w, cudaMemcpyHostToDevice, ctx->stream));
    if (n2) MSC3D_CUDA_TRY(cudaMemcpyAsync(b, twos, n2 * w, cudaMemcpyHostToDevice, ctx->stream));
    MSC3D_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    return MSC3D_OK;
}

int minor(msc3d_ctx* ctx) {
    const Dims& d = ctx->dims;
    const int w = ctx->id_width();
    const cudaStream_t s = ctx->stream;
    const int sms = ctx->num_sms;
    const auto* codes = ctx->ptr<std::uint8_t>("codes");
    const auto* marked = ctx->ptr<std::uint8_t>("marked");
    const std::uint64_t n1 = ctx->count("one_saddles"), n2 = ctx->count("two_saddles");
    const std::uint64_t nde = 3 * d.n_verts;
    // junctions in cell order (saddle_graph.cpp:126-133)
    TRY(msc3d_dev::launch_junction_cells(codes, marked, d, ctx->ws, nullptr, w, ctx->d_small, s, sms, true));
    TRY(ctx->fetch_small(1));
    const std::uint64_t nj = ctx->h_small[0];
    void* jcells = ctx->ensure("junctions", nj, w);
    auto* jlist = static_cast<std::uint32_t*>(ctx->ensure("minor_jlist", nj, 4));
    auto* jidx = static_cast<std::uint32_t*>(ctx->ensure("jidx", nde, 4));
    auto* tmap = static_cast<std::uint32_t*>(ctx->ensure("tmap", nde, 4));
    auto* jdest = static_cast<std::uint32_t*>(ctx->ensure("minor_jdest", 4 * nj, 4));
    auto* sdest = static_cast<std::uint32_t*>(ctx->ensure("minor_sdest", 4 * n1, 4));
    if (!jcells || !jlist || !jidx || !tmap || !jdest || !sdest) return MSC3D_ERR_NOMEM;
    TRY(msc3d_dev::launch_junction_cells(codes, marked, d, ctx->ws, jcells, w, ctx->d_small + 8, s, sms, false));
    if (nj) {
        if (w == 4)
            msc3d_dev::k_junction_dense<std::uint32_t><<<msc3d_dev::grid_for(nj, sms), msc3d_dev::kThreads, 0, s>>>(
                static_cast<const std::uint32_t*>(jcells), nj, d, jlist, jidx);
        else
            msc3d_dev::k_junction_dense<std::uint64_t><<<msc3d_dev::grid_for(nj, sms), msc3d_dev::kThreads, 0, s>>>(
                static_cast<const std::uint64_t*>(jcells), nj, d, jlist, jidx);
        msc3d_dev::count_launch();
    }
    TRY(msc3d_dev::launch_scatter_quad_rank(ctx->ptr<void>("two_saddles"), n2, w, d, tmap, s, sms));
    auto* flags = reinterpret_cast<unsigned int*>(ctx->d_small + 26);
    MSC3D_CUDA_TRY(cudaMemsetAsync(flags, 0, 16, s));
    TRY(msc3d_dev::launch_origin_dests(codes, d, jlist, nullptr, w, nj, jidx, tmap, jdest, nullptr, nullptr, flags,
                                       s, sms));
    TRY(msc3d_dev::launch_origin_dests(codes, d, nullptr, ctx->ptr<void>("one_saddles"), w, n1, jidx, tmap, sdest,
                                       nullptr, nullptr, flags, s, sms));
    TRY(ctx->fetch_small(28));
    if (static_cast<unsigned int>(ctx->h_small[27])) return MSC3D_ERR_RUNTIME;  // saddle_graph.cpp:173-174
    // emit the 4 typed edge lists, each sorted by (src, dst)
    struct Cls {
        const std::uint32_t* dest;
        std::uint64_t n;
        const char* jname;
        const char* tname;
    } cls[2] = {{sdest, n1, "s1_to_j", "s1_to_s2"}, {jdest, nj, "j_to_j", "j_to_s2"}};
    for (const Cls& c : cls) {
        auto* cj = static_cast<std::uint32_t*>(ctx->ensure(std::string(c.jname) + ".cnt", c.n, 4));
        auto* ct = static_cast<std::uint32_t*>(ctx->ensure(std::string(c.tname) + ".cnt", c.n, 4));
        auto* oj = static_cast<std::uint64_t*>(ctx->ensure(std::string(c.jname) + ".off", c.n, 8));
        auto* ot = static_cast<std::uint64_t*>(ctx->ensure(std::string(c.tname) + ".off", c.n, 8));
        if (!cj || !ct || !oj || !ot) return MSC3D_ERR_NOMEM;
        std::uint64_t tj = 0, tt = 0;
        if (c.n) {
            msc3d_dev::k_minor_count<<<msc3d_dev::grid_for(c.n, sms), msc3d_dev::kThreads, 0, s>>>(c.dest, c.n, cj, ct);
            msc3d_dev::count_launch();
            TRY(msc3d_dev::scan_u32(cj, c.n, oj, ctx->d_small, ctx->ws, s));
            TRY(msc3d_dev::scan_u32(ct, c.n, ot, ctx->d_small + 1, ctx->ws2, s));
            TRY(ctx->fetch_small(2));
            tj = ctx->h_small[0];
            tt = ctx->h_small[1];
        }
        auto* js = static_cast<std::uint32_t*>(ctx->ensure(std::string(c.jname) + ".src", tj, 4));
        auto* jd = static_cast<std::uint32_t*>(ctx->ensure(std::string(c.jname) + ".dst", tj, 4));
        auto* jm = static_cast<std::uint64_t*>(ctx->ensure(std::string(c.jname) + ".mult", tj, 8));
        auto* ts = static_cast<std::uint32_t*>(ctx->ensure(std::string(c.tname) + ".src", tt, 4));
        auto* td = static_cast<std::uint32_t*>(ctx->ensure(std::string(c.tname) + ".dst", tt, 4));
        auto* tm = static_cast<std::uint64_t*>(ctx->ensure(std::string(c.tname) + ".mult", tt, 8));
        if (!js || !jd || !jm || !ts || !td || !tm) return MSC3D_ERR_NOMEM;
        if (c.n) {
            msc3d_dev::k_minor_write<<<msc3d_dev::grid_for(c.n, sms), msc3d_dev::kThreads, 0, s>>>(
                c.dest, c.n, oj, ot, js, jd, jm, ts, td, tm);
            msc3d_dev::count_launch();
        }
    }
    MSC3D_CUDA_TRY(cudaGetLastError());
    MSC3D_CUDA_TRY(cudaStreamSynchronize(s));
    return MSC3D_OK;
}

// count_paths on a host DagMinor.  The minor's adjacency (from_edges semantics:
// duplicates summed, zero sums dropped, endpoints validated) and the junction level
// schedule are prepared on the host; every count, product and overflow check runs
// on the device.
int count_minor(msc3d_ctx* ctx, const void* ones, std::uint64_t n1, const void* juncs, std::uint64_t nj,
                const void* twos, std::uint64_t n2, const std::uint32_t* const* src,
                const std::uint32_t* const* dst, const std::uint64_t* const* mult, const std::uint64_t* count,
                int id_width) {
    (void)ones;
    (void)juncs;
    (void)twos;
    (void)id_width;
    const cudaStream_t s = ctx->stream;
    const int sms = ctx->num_sms;
    // ---- host: adjacency in canonical form (path_matrix.cpp:84-113)
    const std::uint64_t rows_of[4] = {n1, nj, nj, n1}, cols_of[4] = {nj, nj, n2, n2};
    std::map<std::pair<std::uint32_t, std::uint32_t>, std::uint64_t> sum[4];
    for (int k = 0; k < 4; ++k)
        for (std::uint64_t i = 0; i < count[k]; ++i) {
            if (src[k][i] >= rows_of[k] || dst[k][i] >= cols_of[k]) return MSC3D_ERR_INVALID;
            std::uint64_t& v = sum[k][{src[k][i], dst[k][i]}];
            if (__builtin_add_overflow(v, mult[k][i], &v)) return MSC3D_ERR_OVERFLOW;
        }
    // junction out-CSR (j_to_j then j_to_s2 per row) and 1-saddle out-CSR
    std::vector<std::vector<std::pair<std::uint32_t, std::uint64_t>>> jout(nj), sout(n1), jpred(nj);
    for (const auto& kv : sum[1])
        if (kv.second) {
            jout[kv.first.first].push_back({kv.first.second, kv.second});
            jpred[kv.first.second].push_back({kv.first.first, kv.second});
        }
    for (const auto& kv : sum[2])
        if (kv.second) jout[kv.first.first].push_back({kv.first.second | msc3d_dev::kTerm, kv.second});
    for (const auto& kv : sum[0])
        if (kv.second) sout[kv.first.first].push_back({kv.first.second, kv.second});
    for (const auto& kv : sum[3])
        if (kv.second) sout[kv.first.first].push_back({kv.first.second | msc3d_dev::kTerm, kv.second});
    auto flatten = [](const std::vector<std::vector<std::pair<std::uint32_t, std::uint64_t>>>& adj,
                      std::vector<std::uint64_t>& off, std::vector<std::uint32_t>& d, std::vector<std::uint64_t>& m) {
        off.assign(adj.size() + 1, 0);
        for (std::size_t i = 0; i < adj.size(); ++i) {
            off[i + 1] = off[i] + adj[i].size();
            for (const auto& e : adj[i]) {
                d.push_back(e.first);
                m.push_back(e.second);
            }
        }
    };
    std::vector<std::uint64_t> joff, soff, poff;
    std::vector<std::uint32_t> jdst, sdst, psrc;
    std::vector<std::uint64_t> jmul, smul, pmul;
    flatten(jout, joff, jdst, jmul);
    flatten(sout, soff, sdst, smul);
    flatten(jpred, poff, psrc, pmul);
    // ---- host: schedule.  Backward levels (sinks first) for P(j); junctions on or
    // upstream of a cycle never become ready.  The reference fails with
    // runtime_error iff such a junction is reachable from a 1-saddle
    // (path_matrix.cpp:201-204).
    std::vector<std::uint32_t> pend(nj);
    for (std::uint64_t j = 0; j < nj; ++j) {
        std::uint32_t c = 0;
        for (const auto& e : jout[j]) c += !(e.first & msc3d_dev::kTerm);
        pend[j] = c;
    }
    std::vector<std::vector<std::uint32_t>> levels;
    std::vector<std::uint32_t> cur;
    for (std::uint32_t j = 0; j < nj; ++j)
        if (!pend[j]) cur.push_back(j);
    std::vector<std::uint8_t> done(nj, 0);
    while (!cur.empty()) {
        std::vector<std::uint32_t> nxt;
        for (const std::uint32_t j : cur) {
            done[j] = 1;
            for (const auto& p : jpred[j])
                if (--pend[p.first] == 0) nxt.push_back(p.first);
        }
        levels.push_back(cur);
        cur.swap(nxt);
    }
    std::vector<std::uint8_t> reach(nj, 0);
    std::vector<std::uint32_t> stack;
    for (std::uint64_t i = 0; i < n1; ++i)
        for (const auto& e : sout[i])
            if (!(e.first & msc3d_dev::kTerm) && !reach[e.first]) {
                reach[e.first] = 1;
                stack.push_back(e.first);
            }
    while (!stack.empty()) {
        const std::uint32_t j = stack.back();
        stack.pop_back();
        for (const auto& e : jout[j])
            if (!(e.first & msc3d_dev::kTerm) && !reach[e.first]) {
                reach[e.first] = 1;
                stack.push_back(e.first);
            }
    }
    for (std::uint64_t j = 0; j < nj; ++j)
        if (reach[j] && !done[j]) return MSC3D_ERR_RUNTIME;
    // forward topological order of the reachable junctions (reverse of the levels)
    std::vector<std::uint32_t> topo;
    for (auto it = levels.rbegin(); it != levels.rend(); ++it)
        for (const std::uint32_t j : *it)
            if (reach[j]) topo.push_back(j);
    std::vector<std::vector<std::uint32_t>> flevels;  // forward levels for the F pass
    {
        std::vector<std::uint32_t> depth(nj, 0);
        std::uint32_t maxd = 0;
        for (const std::uint32_t j : topo) {
            for (const auto& p : jpred[j])
                if (reach[p.first]) depth[j] = std::max(depth[j], depth[p.first] + 1);
            maxd = std::max(maxd, depth[j]);
        }
        flevels.assign(topo.empty() ? 0 : maxd + 1, {});
        for (const std::uint32_t j : topo) flevels[depth[j]].push_back(j);
    }

    // ---- device
    TRY(upload(ctx, "cm_joff", joff));
    TRY(upload(ctx, "cm_jdst", jdst));
    TRY(upload(ctx, "cm_jmul", jmul));
    TRY(upload(ctx, "cm_soff", soff));
    TRY(upload(ctx, "cm_sdst", sdst));
    TRY(upload(ctx, "cm_smul", smul));
    TRY(upload(ctx, "cm_poff", poff));
    TRY(upload(ctx, "cm_psrc", psrc));
    TRY(upload(ctx, "cm_pmul", pmul));
    auto* P_off = static_cast<std::uint64_t*>(ctx->ensure("cm_P_off", std::max<std::uint64_t>(nj, 1), 8));
    auto* P_len = static_cast<std::uint32_t*>(ctx->ensure("cm_P_len", std::max<std::uint64_t>(nj, 1), 4));
    if (!P_off || !P_len) return MSC3D_ERR_NOMEM;
    if (nj) MSC3D_CUDA_TRY(cudaMemsetAsync(P_len, 0, nj * 4, s));
    auto* flags = reinterpret_cast<unsigned int*>(ctx->d_small + 26);
    MSC3D_CUDA_TRY(cudaMemsetAsync(flags, 0, 16, s));
    // pool of all P vectors (grown level by level)
    std::vector<std::uint32_t> host_dummy;
    std::uint64_t pool_n = 0;
    std::uint64_t pool_cap = 1024;
    ctx->ensure("cm_pool_key", pool_cap, 4);
    ctx->ensure("cm_pool_cnt", pool_cap, 8);
    auto grow_pool = [&](std::uint64_t need) -> int {
        if (need <= pool_cap) return MSC3D_OK;
        std::uint64_t cap = std::max(need, 2 * pool_cap);
        void* nk = nullptr;
        void* nc = nullptr;
        if (cudaMalloc(&nk, cap * 4) != cudaSuccess || cudaMalloc(&nc, cap * 8) != cudaSuccess) return MSC3D_ERR_NOMEM;
        if (pool_n) {
            MSC3D_CUDA_TRY(cudaMemcpyAsync(nk, ctx->ptr<void>("cm_pool_key"), pool_n * 4, cudaMemcpyDeviceToDevice, s));
            MSC3D_CUDA_TRY(cudaMemcpyAsync(nc, ctx->ptr<void>("cm_pool_cnt"), pool_n * 8, cudaMemcpyDeviceToDevice, s));
        }
        MSC3D_CUDA_TRY(cudaStreamSynchronize(s));
        DevArray& ak = ctx->arrays["cm_pool_key"];
        DevArray& ac = ctx->arrays["cm_pool_cnt"];
        cudaFree(ak.ptr);
        cudaFree(ac.ptr);
        ak.ptr = nk;
        ak.cap = cap * 4;
        ac.ptr = nc;
        ac.cap = cap * 8;
        pool_cap = cap;
        return MSC3D_OK;
    };
    for (const auto& lvl : levels) {
        const std::uint64_t nr = lvl.size();
        std::vector<std::uint64_t> roff(nr + 1, 0);
        for (std::uint64_t i = 0; i < nr; ++i) roff[i + 1] = roff[i] + jout[lvl[i]].size();
        TRY(upload(ctx, "cm_rows", lvl));
        TRY(upload(ctx, "cm_roff", roff));
        auto* refs = static_cast<Ref*>(ctx->ensure("cm_refs", std::max<std::uint64_t>(roff[nr], 1), sizeof(Ref)));
        if (!refs) return MSC3D_ERR_NOMEM;
        msc3d_dev::k_level_refs<<<msc3d_dev::grid_for(nr, sms), msc3d_dev::kThreads, 0, s>>>(
            ctx->ptr<std::uint32_t>("cm_rows"), nr, ctx->ptr<std::uint64_t>("cm_joff"), ctx->ptr<std::uint32_t>("cm_jdst"),
            ctx->ptr<std::uint64_t>("cm_jmul"), ctx->ptr<std::uint64_t>("cm_roff"), P_off, P_len, refs);
        msc3d_dev::count_launch();
        std::uint64_t produced = 0;
        TRY(merge_rows(ctx, nr, ctx->ptr<std::uint64_t>("cm_roff"), refs, ctx->ptr<std::uint32_t>("cm_pool_key"),
                       ctx->ptr<std::uint64_t>("cm_pool_cnt"), "cm_lvl", &produced));
        TRY(grow_pool(pool_n + produced));
        if (produced) {
            MSC3D_CUDA_TRY(cudaMemcpyAsync(ctx->ptr<std::uint32_t>("cm_pool_key") + pool_n, ctx->ptr<void>("cm_lvl.key"),
                                           produced * 4, cudaMemcpyDeviceToDevice, s));
            MSC3D_CUDA_TRY(cudaMemcpyAsync(ctx->ptr<std::uint64_t>("cm_pool_cnt") + pool_n, ctx->ptr<void>("cm_lvl.cnt"),
                                           produced * 8, cudaMemcpyDeviceToDevice, s));
        }
        msc3d_dev::k_set_rows_P<<<msc3d_dev::grid_for(nr, sms), msc3d_dev::kThreads, 0, s>>>(
            ctx->ptr<std::uint32_t>("cm_rows"), nr, pool_n, ctx->ptr<std::uint64_t>("cm_lvl.off"),
            ctx->ptr<std::uint32_t>("cm_lvl.len"), P_off, P_len);
        msc3d_dev::count_launch();
        pool_n += produced;
    }
    // 1-saddles: rows = all sources, in order
    {
        std::vector<std::uint32_t> rows(n1);
        for (std::uint64_t i = 0; i < n1; ++i) rows[i] = static_cast<std::uint32_t>(i);
        TRY(upload(ctx, "cm_rows", rows));
        auto* refs = static_cast<Ref*>(ctx->ensure("cm_refs", std::max<std::uint64_t>(soff[n1], 1), sizeof(Ref)));
        if (!refs) return MSC3D_ERR_NOMEM;
        if (n1)
            msc3d_dev::k_level_refs<<<msc3d_dev::grid_for(n1, sms), msc3d_dev::kThreads, 0, s>>>(
                ctx->ptr<std::uint32_t>("cm_rows"), n1, ctx->ptr<std::uint64_t>("cm_soff"),
                ctx->ptr<std::uint32_t>("cm_sdst"), ctx->ptr<std::uint64_t>("cm_smul"),
                ctx->ptr<std::uint64_t>("cm_soff"), P_off, P_len, refs);
        msc3d_dev::count_launch();
        std::uint64_t produced = 0;
        TRY(merge_rows(ctx, n1, ctx->ptr<std::uint64_t>("cm_soff"), refs, ctx->ptr<std::uint32_t>("cm_pool_key"),
                       ctx->ptr<std::uint64_t>("cm_pool_cnt"), "cm_src", &produced));
        // expand rows into (one rank, two rank, paths) triples
        std::vector<std::uint32_t> len(n1);
        std::vector<std::uint64_t> off(n1);
        if (n1) {
            MSC3D_CUDA_TRY(cudaMemcpyAsync(len.data(), ctx->ptr<void>("cm_src.len"), n1 * 4, cudaMemcpyDeviceToHost, s));
            MSC3D_CUDA_TRY(cudaMemcpyAsync(off.data(), ctx->ptr<void>("cm_src.off"), n1 * 8, cudaMemcpyDeviceToHost, s));
            MSC3D_CUDA_TRY(cudaStreamSynchronize(s));
        }
        std::vector<std::uint32_t> one(produced);
        for (std::uint64_t i = 0; i < n1; ++i)
            for (std::uint32_t k = 0; k < len[i]; ++k) one[off[i] + k] = static_cast<std::uint32_t>(i);
        TRY(upload(ctx, "ss_one_rank", one));
        void* a = ctx->ensure("ss_two_rank", produced, 4);
        void* b = ctx->ensure("ss_paths", produced, 8);
        if (!a || !b) return MSC3D_ERR_NOMEM;
        if (produced) {
            MSC3D_CUDA_TRY(cudaMemcpyAsync(a, ctx->ptr<void>("cm_src.key"), produced * 4, cudaMemcpyDeviceToDevice, s));
            MSC3D_CUDA_TRY(cudaMemcpyAsync(b, ctx->ptr<void>("cm_src.cnt"), produced * 8, cudaMemcpyDeviceToDevice, s));
        }
    }
    TRY(ctx->fetch_small(27));
    if (ctx->h_small[26] & 0xffffffffu) return MSC3D_ERR_OVERFLOW;
    // A* overflow at junctions no 2-saddle sees (path_matrix.cpp:201-206): forward
    // saturating totals; only when one saturates, the exact per-source check.
    if (!topo.empty()) {
        auto* F = static_cast<std::uint64_t*>(ctx->ensure("cm_F", nj, 8));
        auto* sat = reinterpret_cast<unsigned int*>(ctx->d_small + 62);
        if (!F) return MSC3D_ERR_NOMEM;
        std::vector<std::uint64_t> seed(nj, 0);
        bool seed_sat = false;
        for (std::uint64_t i = 0; i < n1; ++i)
            for (const auto& e : sout[i])
                if (!(e.first & msc3d_dev::kTerm)) {
                    std::uint64_t& v = seed[e.first];
                    if (__builtin_add_overflow(v, e.second, &v)) {
                        v = ~0ull;
                        seed_sat = true;
                    }
                }
        TRY(upload(ctx, "cm_F", seed));
        MSC3D_CUDA_TRY(cudaMemsetAsync(sat, 0, 4, s));
        for (const auto& lvl : flevels) {
            TRY(upload(ctx, "cm_rows", lvl));
            msc3d_dev::k_forward_level<<<msc3d_dev::grid_for(lvl.size(), sms), msc3d_dev::kThreads, 0, s>>>(
                ctx->ptr<std::uint32_t>("cm_rows"), lvl.size(), ctx->ptr<std::uint64_t>("cm_poff"),
                ctx->ptr<std::uint32_t>("cm_psrc"), ctx->ptr<std::uint64_t>("cm_pmul"), F, sat);
            msc3d_dev::count_launch();
        }
        TRY(ctx->fetch_small(63));
        if (seed_sat || static_cast<unsigned int>(ctx->h_small[62])) {
            // dense rows of A* for batches of 1-saddles within a 2 GiB scratch (an overflow
            // verdict for any size, not an allocation failure; slow, but it only runs when
            // some forward total reached 2^64)
            TRY(upload(ctx, "cm_topo", topo));
            std::uint64_t batch = std::max<std::uint64_t>(1, std::min<std::uint64_t>(n1, (1ull << 28) / std::max<std::uint64_t>(nj, 1)));
            if (ctx->exact_batch_rows) batch = std::min(batch, ctx->exact_batch_rows);
            auto* A = static_cast<std::uint64_t*>(ctx->ensure("cm_A", batch * std::max<std::uint64_t>(nj, 1), 8));
            if (!A) return MSC3D_ERR_NOMEM;
            for (std::uint64_t r0 = 0; r0 < n1; r0 += batch) {
                const std::uint64_t nb = std::min(batch, n1 - r0);
                msc3d_dev::k_forward_exact<<<msc3d_dev::grid_for(nb, sms), msc3d_dev::kThreads, 0, s>>>(
                    r0, nb, nj, ctx->ptr<std::uint32_t>("cm_topo"), topo.size(), ctx->ptr<std::uint64_t>("cm_poff"),
                    ctx->ptr<std::uint32_t>("cm_psrc"), ctx->ptr<std::uint64_t>("cm_pmul"),
                    ctx->ptr<std::uint64_t>("cm_soff"), ctx->ptr<std::uint32_t>("cm_sdst"),
                    ctx->ptr<std::uint64_t>("cm_smul"), A, flags);
                msc3d_dev::count_launch();
                TRY(ctx->fetch_small(27));
                if (ctx->h_small[26] & 0xffffffffu) return MSC3D_ERR_OVERFLOW;
            }
        }
    }
    MSC3D_CUDA_TRY(cudaStreamSynchronize(s));
    return MSC3D_OK;
}

int sp_op(msc3d_ctx* ctx, int op, std::uint32_t xr, std::uint32_t xc, const std::uint64_t* xp,
          const std::uint32_t* xcol, const std::uint64_t* xcnt, std::uint32_t yr, std::uint32_t yc,
          const std::uint64_t* yp, const std::uint32_t* ycol, const std::uint64_t* ycnt) {
    if (op == 0 && xc != yr) return MSC3D_ERR_INVALID;
    if (op == 1 && (xr != yr || xc != yc)) return MSC3D_ERR_INVALID;
    const cudaStream_t s = ctx->stream;
    const int sms = ctx->num_sms;
    const std::uint64_t nx = xp[xr], ny = yp[yr];
    // pool = x entries ++ y entries
    std::vector<std::uint32_t> key(nx + ny);
    std::vector<std::uint64_t> cnt(nx + ny);
    for (std::uint64_t i = 0; i < nx; ++i) {
        key[i] = xcol[i];
        cnt[i] = xcnt[i];
    }
    for (std::uint64_t i = 0; i < ny; ++i) {
        key[nx + i] = ycol[i];
        cnt[nx + i] = ycnt[i];
    }
    TRY(upload(ctx, "sp_pool_key", key));
    TRY(upload(ctx, "sp_pool_cnt", cnt));
    TRY(upload(ctx, "sp_xp", std::vector<std::uint64_t>(xp, xp + xr + 1)));
    TRY(upload(ctx, "sp_xc", std::vector<std::uint32_t>(xcol, xcol + nx)));
    TRY(upload(ctx, "sp_xv", std::vector<std::uint64_t>(xcnt, xcnt + nx)));
    TRY(upload(ctx, "sp_yp", std::vector<std::uint64_t>(yp, yp + yr + 1)));
    std::vector<std::uint64_t> roff(xr + 1, 0);
    for (std::uint32_t r = 0; r < xr; ++r) roff[r + 1] = roff[r] + (op == 0 ? xp[r + 1] - xp[r] : 2);
    TRY(upload(ctx, "sp_roff", roff));
    auto* refs = static_cast<Ref*>(ctx->ensure("sp_refs", std::max<std::uint64_t>(roff[xr], 1), sizeof(Ref)));
    if (!refs) return MSC3D_ERR_NOMEM;
    auto* flags = reinterpret_cast<unsigned int*>(ctx->d_small + 26);
    MSC3D_CUDA_TRY(cudaMemsetAsync(flags, 0, 16, s));
    if (xr) {
        msc3d_dev::k_sp_refs<<<msc3d_dev::grid_for(xr, sms), msc3d_dev::kThreads, 0, s>>>(
            op, xr, ctx->ptr<std::uint64_t>("sp_xp"), ctx->ptr<std::uint32_t>("sp_xc"), ctx->ptr<std::uint64_t>("sp_xv"),
            ctx->ptr<std::uint64_t>("sp_yp"), nx, ctx->ptr<std::uint64_t>("sp_roff"), refs);
        msc3d_dev::count_launch();
    }
    std::uint64_t produced = 0;
    TRY(merge_rows(ctx, xr, ctx->ptr<std::uint64_t>("sp_roff"), refs, ctx->ptr<std::uint32_t>("sp_pool_key"),
                   ctx->ptr<std::uint64_t>("sp_pool_cnt"), "sp_out", &produced));
    TRY(ctx->fetch_small(27));
    if (ctx->h_small[26] & 0xffffffffu) return MSC3D_ERR_OVERFLOW;
    // row_ptr = [offsets..., total]
    auto* rp = static_cast<std::uint64_t*>(ctx->ensure("sp_row_ptr", static_cast<std::uint64_t>(xr) + 1, 8));
    if (!rp) return MSC3D_ERR_NOMEM;
    if (xr) MSC3D_CUDA_TRY(cudaMemcpyAsync(rp, ctx->ptr<void>("sp_out.off"), xr * 8ull, cudaMemcpyDeviceToDevice, s));
    ctx->h_small[63] = produced;
    MSC3D_CUDA_TRY(cudaMemcpyAsync(rp + xr, &ctx->h_small[63], 8, cudaMemcpyHostToDevice, s));
    void* ci = ctx->ensure("sp_col_idx", produced, 4);
    void* cv = ctx->ensure("sp_count", produced, 8);
    if (!ci || !cv) return MSC3D_ERR_NOMEM;
    if (produced) {
        MSC3D_CUDA_TRY(cudaMemcpyAsync(ci, ctx->ptr<void>("sp_out.key"), produced * 4, cudaMemcpyDeviceToDevice, s));
        MSC3D_CUDA_TRY(cudaMemcpyAsync(cv, ctx->ptr<void>("sp_out.cnt"), produced * 8, cudaMemcpyDeviceToDevice, s));
    }
    MSC3D_CUDA_TRY(cudaStreamSynchronize(s));
    return MSC3D_OK;
}

}  // namespace msc3d_stage

// Host-side launch wrappers for every device stage (implemented in the .cu files).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"

namespace msc3d_dev {

// One growable scratch buffer (single outstanding use).  Owned by the context.
struct Workspace {
    void* ptr = nullptr;
    std::size_t cap = 0;
    void* get(std::size_t bytes) {
        if (bytes <= cap && ptr) return ptr;
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        cap = 0;
        const std::size_t want = bytes + bytes / 4 + 4096;
        if (cudaMalloc(&ptr, want) != cudaSuccess) return nullptr;
        cap = want;
        return ptr;
    }
    ~Workspace() {
        if (ptr) cudaFree(ptr);
    }
};

// gradient.cu
int launch_gradient(const void* values, int value_type, const Dims& d, std::uint8_t* codes,
                    std::uint32_t* parent0, std::uint32_t* parent3, cudaStream_t stream,
                    unsigned long long* crit_totals, std::uint32_t* const lists3[3],
                    unsigned long long* list_counts, int num_sms);

// The gradient in pieces (streamed input): tables + counters; tile layers
// [tz0, tz1) (TZ = 2 vertex planes each; they read vertex planes up to
// gradient_layer_last_plane(d, tz1)); the large-star list kernels.
int gradient_begin(unsigned long long* crit_totals, unsigned long long* list_counts, cudaStream_t stream);
unsigned gradient_tile_layers(const Dims& d);
int gradient_layer_last_plane(const Dims& d, unsigned tz_end);
int gradient_tiles(const void* values, int value_type, const Dims& d, std::uint8_t* codes, std::uint32_t* parent0,
                   std::uint32_t* parent3, cudaStream_t stream, unsigned long long* crit_totals,
                   std::uint32_t* const lists3[3], unsigned long long* list_counts, int num_sms, unsigned tz0,
                   unsigned tz1);
int gradient_finish(const void* values, int value_type, const Dims& d, std::uint8_t* codes, std::uint32_t* parent0,
                    std::uint32_t* parent3, cudaStream_t stream, unsigned long long* crit_totals,
                    std::uint32_t* const lists3[3], unsigned long long* list_counts, int num_sms);

// critical.cu
int launch_critical_count(const std::uint8_t* codes, const Dims& d, std::uint64_t* d_totals,
                          cudaStream_t s, int num_sms);
// validate_gradient's matching audit; *bad (zeroed by the caller) counts violations
int launch_critical_compact(const std::uint8_t* codes, const Dims& d, Workspace& ws,
                            void* const outs[4], int id_width, std::uint64_t* d_totals,
                            cudaStream_t s);
int launch_saddle_count(const std::uint8_t* codes, const Dims& d, std::uint64_t* d_totals,
                        cudaStream_t s, int num_sms);
int launch_saddle_compact(const std::uint8_t* codes, const Dims& d, Workspace& ws, void* out,
                          int id_width, std::uint64_t* d_totals, cudaStream_t s);
int launch_junction_cells(const std::uint8_t* codes, const std::uint8_t* marked, const Dims& d,
                          Workspace& ws, void* out, int id_width, std::uint64_t* d_totals,
                          cudaStream_t s, int num_sms, bool count_only);
int launch_marked_critical_count(const std::uint8_t* codes, const std::uint8_t* marked,
                                 const Dims& d, std::uint64_t* d_totals, cudaStream_t s,
                                 int num_sms);
int launch_marked_critical_compact(const std::uint8_t* codes, const std::uint8_t* marked,
                                   const Dims& d, Workspace& ws, void* const outs[4],
                                   int id_width, std::uint64_t* d_totals, cudaStream_t s);

}  // namespace msc3d_dev

namespace msc3d_dev {
// primitives.cu
// Copy n u64 device -> mapped host memory with a kernel (no copy engine).
int launch_small_copy(const std::uint64_t* src, std::uint64_t* dst_mapped, int n, cudaStream_t s);
// *first_bad = min(*first_bad, index of a non-finite sample) (grid.cpp:86-88)
int launch_check_finite(const void* values, int value_type, std::uint64_t n, unsigned long long* first_bad,
                        cudaStream_t s, int num_sms);
int scan_u32(const std::uint32_t* in, std::uint64_t n, std::uint64_t* out, std::uint64_t* d_total,
             Workspace& ws, cudaStream_t s);

// extrema.cu
int launch_forest(const std::uint8_t* codes, const Dims& d, int dim, std::uint32_t* parent,
                  cudaStream_t s, int num_sms);
int launch_double_round(const std::uint32_t* in, std::uint32_t* out, std::uint64_t n,
                        unsigned int* changed, cudaStream_t s, int num_sms);
// roots of both extremum forests in place, all rounds in one cooperative launch;
// conv: (n0 + n3 + 31) / 32 words of scratch
// Tile-local root pre-resolution of a lattice-neighbour forest over a gx*gy*gz grid
// (every parent then points at its root or out of its box); then launch_jump_all.
// skip (optional): the jump mask over the concatenated index space (item k = kofs + j),
// in which every exit target's bit is cleared; launch_jump_all(..., masked = 1) then
// resolves only those, launch_resolve_exits the rest.
int launch_tile_roots(std::uint32_t* p, std::uint64_t gx, std::uint64_t gy, std::uint64_t gz, unsigned int* skip,
                      std::uint64_t kofs, unsigned int* cycle, cudaStream_t s);
int launch_resolve_exits(std::uint32_t* p0, std::uint64_t n0, std::uint32_t* p3, std::uint64_t n3, cudaStream_t s,
                         int num_sms);
int launch_jump_all(std::uint32_t* p0, std::uint64_t n0, std::uint32_t* p3, std::uint64_t n3, unsigned int* conv,
                    unsigned int* flags,
                    unsigned long long* rounds, cudaStream_t s, int num_sms, int masked = 0);
// rank: nwords uint2 {rank of the word's first set bit, bits} over dense(crit[k]);
// bits / cnt / pre: nwords scratch (u32, u32, u64)
int launch_rank_map(const void* crit, std::uint64_t n, int id_width, const Dims& d, int dim,
                    unsigned int* bits, std::uint32_t* cnt, std::uint64_t* pre, void* rank, std::uint64_t nwords,
                    Workspace& ws, std::uint64_t* d_total, cudaStream_t s, int num_sms);
int launch_gather(const std::uint32_t* label, RankRemap remap, std::uint64_t n,
                  std::uint32_t* out, cudaStream_t s, int num_sms);
int launch_se_slots(const std::uint8_t* codes, const Dims& d, const void* saddles,
                    std::uint64_t ns, int id_width, const std::uint32_t* l0,
                    const std::uint32_t* l3, std::uint64_t* slot, std::uint32_t* cnt,
                    cudaStream_t s, int num_sms);
int launch_se_write(const void* saddles, std::uint64_t ns, int id_width,
                    const std::uint64_t* slot, const std::uint64_t* off, void* out_s, void* out_e,
                    std::uint32_t* out_m, cudaStream_t s, int num_sms);
}  // namespace msc3d_dev

namespace msc3d_dev {
// saddle.cu
int launch_bfs_sources(const std::uint8_t* codes, const Dims& d, const void* src, std::uint64_t n,
                       int id_width, unsigned int* bitmap, std::uint32_t* frontier, unsigned int* bad,
                       cudaStream_t s, int num_sms);
int launch_marked_bytes(const std::uint8_t* codes, const Dims& d, const unsigned int* bitmap,
                        std::uint64_t nwords, std::uint8_t* marked, cudaStream_t s, int num_sms);
int launch_scatter_quad_rank(const void* list, std::uint64_t n, int id_width, const Dims& d,
                             std::uint32_t* tmap, cudaStream_t s, int num_sms);
int launch_origin_dests(const std::uint8_t* codes, const Dims& d, const std::uint32_t* jlist,
                        const void* srcs, int id_width, std::uint64_t n, const std::uint32_t* jidx,
                        const std::uint32_t* tmap, std::uint32_t* dest, std::uint32_t* pending,
                        std::uint32_t* indeg, unsigned int* flags, cudaStream_t s, int num_sms);
}  // namespace msc3d_dev

namespace msc3d_dev {
// assemble.cu
int launch_gather_ids(const void* list, const std::uint32_t* idx, std::uint64_t n, int id_width,
                      void* out, cudaStream_t s, int num_sms);
// CriticalPoint::value of every critical cell (max vertex by value, then id), as f64
int launch_cp_values(const void* cells, int id_width, std::uint64_t n, const Dims& d, const void* values,
                     int value_type, double* out, cudaStream_t s, int num_sms);
int launch_cp_concat(const void* src, std::uint64_t n, std::uint64_t at, int index, int id_width,
                     void* cp_cell, std::uint8_t* cp_index, cudaStream_t s, int num_sms);
int launch_arcs_min(const void* crit1, std::uint64_t n1, int id_width, const Dims& d,
                    const std::uint32_t* label0, RankRemap remap0, std::uint32_t base1,
                    std::uint32_t* slot_min, std::uint32_t* per_min, cudaStream_t s, int num_sms);
int launch_arcs_min_sort(const std::uint32_t* slot_min, std::uint64_t n1, std::uint32_t base1,
                         const std::uint64_t* off, std::uint64_t n0, std::uint64_t total,
                         std::uint32_t* cursor, std::uint64_t* key, std::uint64_t* scratch,
                         std::uint32_t* large, unsigned long long* n_large,
                         std::uint64_t* h_small, std::uint32_t* asrc, std::uint32_t* adst,
                         std::uint64_t* amult, cudaStream_t s, int num_sms);
int launch_bucket_sort(const std::uint64_t* off, std::uint64_t nb, std::uint64_t total,
                       std::uint64_t* key, std::uint64_t* scratch, std::uint32_t* large,
                       unsigned long long* n_large, std::uint64_t* h_small, cudaStream_t s, int num_sms);
int launch_arcs_max(const void* crit2, std::uint64_t n2, int id_width, const Dims& d,
                    const std::uint32_t* label3, RankRemap remap3, std::uint32_t* slot,
                    std::uint32_t* cnt, cudaStream_t s, int num_sms);
// multiplicities for the host: one byte each (255 = escaped) + (index, value) escapes
int launch_pack_mult(const std::uint64_t* mult, std::uint64_t n, std::uint64_t vmax, std::uint8_t* out8, void* esc,
                     std::uint64_t cap, unsigned long long* n_esc, cudaStream_t s, int num_sms);
// sorted u32 values for the host: byte deltas (255 = escaped absolute value) + a u32
// head per src_chunk() entries
int launch_pack_src(const std::uint32_t* src, std::uint64_t n, std::uint64_t vmax, std::uint8_t* out8,
                    std::uint32_t* heads, void* esc, std::uint64_t cap, unsigned long long* n_esc, cudaStream_t s,
                    int num_sms);
std::uint64_t src_chunk();
int launch_arcs_max_emit(const std::uint32_t* slot, std::uint64_t n2, std::uint32_t base2,
                         const std::uint64_t* off, std::uint32_t* asrc, std::uint32_t* adst,
                         std::uint64_t* amult, cudaStream_t s, int num_sms);
}  // namespace msc3d_dev

namespace msc3d_dev {
// dag.cu -- successor table, reachability, junction ranks, branch walks, counting
struct CountLaunch {
    const void* node;               // node_rec_bytes() per node: nj junctions, then n1 1-saddles
    std::uint8_t* pending;          // one byte per node
    const std::uint8_t* pending0;
    const std::uint32_t* rsrc;      // parents beyond the inline ones
    void* rec;                      // count_rec_bytes() per junction
    std::uint32_t* pool_key;
    std::uint64_t* pool_cnt;
    unsigned long long* pool_top;   // count_arenas() counters
    std::uint64_t arena_cap;
    std::uint32_t* slen;
    std::uint64_t nj, n1;
    std::uint32_t* fa;              // frontier buffers (nj + n1 each)
    std::uint32_t* fb;
    unsigned long long* cnt;        // 3 counters
    unsigned long long* stats;      // [0] rounds
    unsigned long long* done;
    unsigned int* flags;            // [0] overflow [1] pool exhausted
    unsigned long long* diag;       // optional development diagnostics (nullptr: off)
    std::uint32_t* heavy_q;         // capacity nj + n1
    unsigned long long* heavy_n;    // 2 counters, zeroed (count_write's heavy queue)
    const void* dest;               // uint4 branch destinations per node (junctions, then 1-saddles)
    const std::uint32_t* ready;     // junctions without pending children (Kahn's round 0)
    const unsigned long long* n_ready;
    unsigned long long* heavy_rounds;  // 6 counters, zeroed (Kahn rounds' heavy queues: size, head x 3)
    unsigned long long* resume;     // 3 words of state between the two configurations
    const std::uint32_t* indeg;     // parents per junction
    const std::uint64_t* ovoff;     // overflow-list offsets
    unsigned long long switch_below;  // frontier size below which the tail configuration runs
    bool async_tail = false;          // the tail without rounds (k_count_async)
    const unsigned long long* n_skip = nullptr;     // contracted junctions (async tail's total)
    const unsigned long long* n_predone = nullptr;  // junctions finished by the walks
    unsigned long long* qctl = nullptr;  // async tail: head / tail / done, 128 bytes apart (48 words)
};
int count_rec_bytes();
int count_arenas();
int launch_succ_table(const std::uint8_t* codes, const Dims& d, std::uint16_t* succ, cudaStream_t s, int num_sms);
int launch_reach(const std::uint16_t* succ, const Dims& d, unsigned int* bitmap, std::uint32_t* fa,
                 std::uint32_t* fb, unsigned long long cap, unsigned long long* cnt, unsigned long long* stats,
                 cudaStream_t s, int num_sms);
int launch_junction_bits(const std::uint16_t* succ, const unsigned int* bitmap, std::uint64_t nwords,
                         unsigned int* jbits, std::uint32_t* jcnt, unsigned long long* nodes, cudaStream_t s,
                         int num_sms);
// jrank: nwords uint2 (first rank of the word, its junction bits)
int launch_junction_list(const unsigned int* jbits, std::uint64_t nwords, const std::uint64_t* woff, void* jrank,
                         std::uint32_t* jlist, cudaStream_t s, int num_sms);
// junction launch: rec / predone (bit per junction) / n_predone set, slen null;
// 1-saddle launch: slen set (their merged length when all branches are terminal), rec/predone null
// rank words of the sorted 2-saddle list by cell id (n_cells / 32 + 1 uint2)
int launch_term_rank(const void* list, std::uint64_t n, int id_width, std::uint64_t n_cells, void* trank,
                     cudaStream_t s, int num_sms);
int launch_walk(const std::uint16_t* succ, const Dims& d, const void* jrank,
                const std::uint32_t* tmap, const void* trank, const std::uint32_t* jlist, const void* srcs, int id_width,
                std::uint64_t n, void* node, std::uint8_t* pending, unsigned int* flags, void* rec,
                std::uint32_t* slen, unsigned int* predone, unsigned long long* n_predone, std::uint32_t* fwd,
                unsigned int* ptbits, cudaStream_t s,
                int num_sms);
int node_rec_bytes();

int launch_rewrite(void* node, void* dest, std::uint64_t nj, std::uint64_t n_nodes, const std::uint32_t* fwd,
                   const unsigned int* ptbits, const unsigned int* predone, std::uint8_t* pending, std::uint32_t* indeg, void* ovq, unsigned long long* ovq_n,
                   std::uint64_t ovq_cap, unsigned long long* n_skip, std::uint32_t* ready,
                   unsigned long long* n_ready, cudaStream_t s, int num_sms);
int launch_parent_overflow(const std::uint32_t* indeg, std::uint64_t nj, std::uint64_t* ovoff,
                           unsigned long long* total, cudaStream_t s, int num_sms);
// node records' parent counts / overflow offsets, and the queued overflow parents
int launch_fill_parents(void* node, std::uint64_t nj, const std::uint32_t* indeg, const std::uint64_t* ovoff,
                        const void* ovq, std::uint64_t n_ovq, std::uint32_t* rsrc, cudaStream_t s, int num_sms);
int launch_count(const CountLaunch& L, cudaStream_t s, int num_sms);
// merged lengths of the 1-saddles the walk did not finish (after k_count) -> L.slen
int launch_source_len(const CountLaunch& L, cudaStream_t s, int num_sms);
int launch_count_write(const CountLaunch& L, const std::uint64_t* off, std::uint32_t* o_one, std::uint32_t* o_two,
                       std::uint64_t* o_cnt, std::uint32_t base_one, std::uint32_t base_two, cudaStream_t s,
                       int num_sms);
}  // namespace msc3d_dev

/*
 * msc3d_cuda.h -- the C ABI of the B200 Morse-Smale-complex pipeline.
 *
 * This is the drop-in boundary under the reference library's public C++ API
 * (/root/reference/proj/include/msc3d/*.hpp).  The reference has no FFI of its
 * own; its "operator API" is those headers.  Our C++ layer
 * (paper_2009_03707_b200/csrc/msc3d_api.cpp, header include/msc3d/api.hpp)
 * keeps the reference's signatures and calls the functions below; Python (ctypes)
 * calls them directly.  No C++ or torch types cross this boundary: plain
 * pointers, sizes, int status codes.  No exceptions cross it either: the C++
 * wrappers turn the status codes back into the reference's exception types
 * (see msc3d_status_string).
 *
 * Conventions
 *   - Lattice / cell ids / pair codes exactly as grid.hpp:8-23, gradient.hpp:29-41.
 *   - Cell-id arrays are uint32 when the lattice has < 2^32 cells (the reference's
 *     CellIndex, grid.hpp:33) and uint64 above that (configs 4-5; the reference
 *     rejects those grids, grid.cpp:17-20).  msc3d_id_width() says which.
 *   - Dense vertex / cube indices (parents, labels) are uint32 (requires
 *     nx*ny*nz < 2^32).
 *   - Every stage runs on the context's CUDA stream; results stay in device
 *     memory owned by the context until downloaded.
 *   - Results are identical for every run and every device count (the reference's
 *     "any thread count" determinism, primitives.hpp:3-8).
 */
#ifndef MSC3D_CUDA_H
#define MSC3D_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (the reference's exception types, msc3d_cli.cpp:157-166) ---- */
#define MSC3D_OK 0
#define MSC3D_ERR_INVALID 1  /* std::invalid_argument (bad dims, non-finite value, bad source) */
#define MSC3D_ERR_OVERFLOW 2 /* std::overflow_error   (path count leaves 64 bits, path_matrix.cpp:44-48) */
#define MSC3D_ERR_RUNTIME 3  /* std::runtime_error    (cycle guards saddle_graph.cpp:173, path_matrix.cpp:202) */
#define MSC3D_ERR_CUDA 4     /* CUDA runtime failure / no device */
#define MSC3D_ERR_NOMEM 5    /* device allocation failed */
#define MSC3D_ERR_IO 6       /* IoError (volume.hpp:22-25) */
#define MSC3D_ERR_STATE 7    /* a stage was called before its inputs exist */

#define MSC3D_VALUE_F32 0
#define MSC3D_VALUE_F64 1

typedef struct msc3d_dims {
    int64_t nx, ny, nz; /* vertices per axis, each >= 2 (grid.cpp:13-16) */
} msc3d_dims;

typedef struct msc3d_ctx msc3d_ctx;

const char* msc3d_status_string(int status);
/* 0 ok / MSC3D_ERR_INVALID for dims < 2; allow_wide = 0 also rejects > 2^32-1 cells
 * exactly like GridDims::GridDims (grid.cpp:11-21). */
int msc3d_check_dims(msc3d_dims d, int allow_wide);
int msc3d_id_width(msc3d_dims d); /* 4 or 8 */
uint64_t msc3d_total_cells(msc3d_dims d);

/* ---- context ------------------------------------------------------------------------ */
int msc3d_ctx_create(msc3d_ctx** out, int device);
void msc3d_ctx_destroy(msc3d_ctx* ctx);
/* cudaStream_t passed as void*; NULL = the context's own non-blocking stream. */
int msc3d_ctx_set_stream(msc3d_ctx* ctx, void* stream);
void* msc3d_ctx_stream(msc3d_ctx* ctx);
int msc3d_ctx_sync(msc3d_ctx* ctx);
/* Number of kernels this context launched since creation (bench evidence). */
uint64_t msc3d_ctx_launches(msc3d_ctx* ctx);

/* Named device arrays owned by the context ("codes", "crit1", "labels_min", ...).
 * *elem_bytes is the element width; *count the number of elements. */
int msc3d_ctx_array(msc3d_ctx* ctx, const char* name, void** device_ptr, uint64_t* count,
                    int* elem_bytes);
/* After a compute: "cp_value" (f64 per critical point) = the sample at the cell's
 * maximum vertex (larger value, then larger id; grid.cpp:129-137) -- CriticalPoint::value
 * of msc.cpp:106 -- from "cp_cell" and the bound samples. */
int msc3d_ctx_cp_values(msc3d_ctx* ctx);

/* Page-locked host memory for the host-buffer entry points (full-bandwidth copies). */
int msc3d_host_alloc(void** out, uint64_t bytes);
void msc3d_host_free(void* p);

/* Copy a named array to host memory (capacity in bytes); synchronises the stream. */
int msc3d_ctx_download(msc3d_ctx* ctx, const char* name, void* host, uint64_t capacity_bytes);
/* Context options (not in the reference; defaults reproduce it exactly):
 *   "wide_ids" (0/1)          64-bit cell-id lists on any grid -- the layout grids with
 *                             >= 2^32 cells use (configs 4-5), testable on small grids;
 *   "exact_batch_rows" (>=0)  1-saddles per batch of the exact A* overflow check
 *                             (0 = as many as 2 GiB of dense rows hold);
 *   "kahn_switch_below" (>=1) frontier size at which path counting leaves its wide
 *                             launch configuration for the tail one (default 2^18);
 *   "side_stream" (0/1)       assemble the extremum-side outputs on a second stream,
 *                             beside the saddle stages (default 0);
 *   "kahn_async" (0/1)        path counting's tail without rounds (default 1; 0: the
 *                             round-based tail configuration);
 *   "frontier_cap" (>=0)      initial entries of the BFS frontier buffers (0 = 4 x the
 *                             sources; a level that does not fit reruns the BFS with
 *                             buffers of every dense edge);
 *   "term_rank_words" (0/1)   the walks' 2-saddle rank lookup grids above 2^28 vertices
 *                             use (rank words in cell order), on any grid;
 *   "release_transients" (-1/0/1) free each stage's scratch arrays once they are dead:
 *                             1 on any grid, 0 never, -1 (default) above 2^32 cells when
 *                             the saddle stages may not fit beside them (1 KB per saddle
 *                             against the free device memory);
 *   "d2h_narrow" (0/1)        host deliveries send multiplicities as one byte per arc
 *                             plus an escape list, widened by host threads (default 1);
 *   "d2h_escape_cap" (>=0)    escape entries per arc block (0 = n/16 + 1024; more
 *                             escapes -> the u64 array is copied instead);
 *   "d2h_narrow_max" (0..254) largest multiplicity / source step sent as its byte
 *                             (default 254; tests lower it to exercise the escapes).
 * Unknown names / bad values -> MSC3D_ERR_INVALID. */
int msc3d_ctx_set_option(msc3d_ctx* ctx, const char* name, int64_t value);
/* Scalar results ("rounds0", "rounds3", "euler", "bfs_levels", ...); also
 * "device_bytes_held" / "device_bytes_peak": device memory of the context's arrays now /
 * at its high-water mark. */
int msc3d_ctx_scalar(msc3d_ctx* ctx, const char* name, int64_t* value);

/* ---- scalar-grid load: ScalarField / read_volume (grid.hpp:117-125, volume.hpp:42) -- */
/* Upload samples (host pointer; f32 or f64 x-fastest) and validate them on device:
 * non-finite -> MSC3D_ERR_INVALID (grid.cpp:86-88). */
int msc3d_ctx_load_values(msc3d_ctx* ctx, msc3d_dims dims, int value_type, const void* host_values);
/* Same from a device pointer (not copied; must outlive the context's use of it). */
int msc3d_ctx_bind_values(msc3d_ctx* ctx, msc3d_dims dims, int value_type, const void* device_values);
/* Raw volume file -> device f32/f64 (u8/u16 widen exactly to f32), volume.cpp:67-96.
 * dtype "u8"|"u16"|"f32"|"f64". */
int msc3d_ctx_read_volume(msc3d_ctx* ctx, const char* path, msc3d_dims dims, const char* dtype,
                          int big_endian);

/* ---- gradient: assign_gradient (gradient.hpp:66) -> array "codes" (u8, N) ------------ */
int msc3d_ctx_gradient(msc3d_ctx* ctx);
/* Install an existing GradientField (host codes) for the stage entry points below. */
int msc3d_ctx_load_codes(msc3d_ctx* ctx, msc3d_dims dims, const uint8_t* host_codes);

/* Install a GradientField already in device memory (copied; e.g. assembled from
 * z-slabs computed on several GPUs). */
int msc3d_ctx_bind_codes(msc3d_ctx* ctx, msc3d_dims dims, const uint8_t* device_codes);

/* ---- critical cells: extract_critical_cells (gradient.hpp:80) -> "crit0".."crit3" --- */
int msc3d_ctx_critical(msc3d_ctx* ctx);

/* ---- manifold traversal (extrema.hpp:43-78) ------------------------------------------ */
/* build_forest -> "parent0" (u32, V) or "parent3" (u32, Cu). */
int msc3d_ctx_forest(msc3d_ctx* ctx, int dim);
/* find_roots: synchronous pointer doubling, bit-exact labels and round count
 * (extrema.cpp:79-101) -> "label0"/"label3", scalar "rounds0"/"rounds3". */
int msc3d_ctx_roots(msc3d_ctx* ctx, int dim);
/* Install a parent array (host) for find_roots on arbitrary forests. */
int msc3d_ctx_load_parent(msc3d_ctx* ctx, int dim, const uint32_t* host_parent, uint64_t n);
/* saddle_extremum_arcs (extrema.cpp:103-148) from "label0"/"label3"
 * -> "se_saddle" (id), "se_extremum" (id), "se_mult" (u32), reference order. */
int msc3d_ctx_se_arcs(msc3d_ctx* ctx);
int msc3d_ctx_load_labels(msc3d_ctx* ctx, const uint32_t* host_label0, const uint32_t* host_label3);

/* ---- audits (gradient.cpp:299-377, msc.cpp:149-167), all on the device ------------------ */
/* validate_gradient of the context's codes: out = {matching_violations,
 * cells_in_closed_vpath, acyclicity_checked, degenerate} (GradientReport,
 * gradient.hpp:83-91); the acyclicity (Kahn peeling of the V-path relation) runs only
 * when the lattice has <= max_cells_for_cycles cells, as the reference.  Offending cells
 * (up to 4096) in array "audit_samples". */
int msc3d_ctx_validate_gradient(msc3d_ctx* ctx, uint64_t max_cells_for_cycles, uint64_t out[4]);
/* boundary_check of the last compute's complex ("cp_index", "arc_*"): *n_odd odd
 * (top, low) pairs in "odd_top" / "odd_low" (u32 cp ids), ordered by top, then low. */
int msc3d_ctx_boundary_check(msc3d_ctx* ctx, uint64_t* n_odd);
/* The same on a complex given as host arrays (cp_index per critical point, arcs). */
int msc3d_boundary_check_host(msc3d_ctx* ctx, uint64_t n_cp, const uint8_t* cp_index, uint64_t n_arcs,
                              const uint32_t* src, const uint32_t* dst, const uint64_t* mult, uint64_t* n_odd);

/* ---- saddle graph (saddle_graph.hpp:39-74) ------------------------------------------- */
/* mark_reachable from the given 1-saddles (host ids, width msc3d_id_width); NULL/0 =
 * all critical 1-cells.  -> "marked" (u8, N), "one_saddles", "two_saddles". */
int msc3d_ctx_mark(msc3d_ctx* ctx, const void* host_sources, uint64_t n_sources);
/* Install a MarkedSubgraph (host marked bytes + ascending 1-/2-saddle ids) for
 * build_minor (saddle_graph.hpp:45-50). */
int msc3d_ctx_load_marked(msc3d_ctx* ctx, const uint8_t* host_marked, const void* one_saddles,
                          uint64_t n1, const void* two_saddles, uint64_t n2);
/* build_minor -> "junctions" + 4 typed edge lists "<kind>.src/.dst" (u32) ".mult" (u64),
 * kind in s1_to_j, j_to_j, j_to_s2, s1_to_s2 (saddle_graph.cpp:121-217). */
int msc3d_ctx_minor(msc3d_ctx* ctx);

/* ---- path counting (path_matrix.hpp:40-64) ------------------------------------------- */
/* count_paths on the device DAG (after msc3d_ctx_mark): branch walks to the ends of
 * junction-free chains, then sparse count vectors over the junction graph in reverse
 * topological order (Kahn rounds in one cooperative kernel) -> "ss_one", "ss_two"
 * (ids), "ss_paths" (u64), sorted by (one, two).  MSC3D_ERR_OVERFLOW with the
 * reference's semantics. */
int msc3d_ctx_count(msc3d_ctx* ctx);
/* count_paths on an explicit DagMinor (host arrays; edge lists in the order
 * s1_to_j, j_to_j, j_to_s2, s1_to_s2) -> "ss_one", "ss_two", "ss_paths". */
int msc3d_ctx_count_minor(msc3d_ctx* ctx, const void* one_saddles, uint64_t n1,
                          const void* junctions, uint64_t nj, const void* two_saddles,
                          uint64_t n2, const uint32_t* const* src, const uint32_t* const* dst,
                          const uint64_t* const* mult, const uint64_t* count, int id_width);

/* sp_multiply (op 0) / sp_add (op 1) of two canonical CSR count matrices
 * (path_matrix.hpp:40-52, path_matrix.cpp:115-186) -> "sp_row_ptr" (u64, rows+1),
 * "sp_col_idx" (u32), "sp_count" (u64).  MSC3D_ERR_OVERFLOW as the reference. */
int msc3d_sp_op(msc3d_ctx* ctx, int op, uint32_t x_rows, uint32_t x_cols, const uint64_t* x_row_ptr,
                const uint32_t* x_col_idx, const uint64_t* x_count, uint32_t y_rows, uint32_t y_cols,
                const uint64_t* y_row_ptr, const uint32_t* y_col_idx, const uint64_t* y_count);

/* ---- MS graph: compute (msc.hpp:87) ----------------------------------------------------- */
#define MSC3D_OPT_SEGMENTATION 1 /* ComputeOptions::with_segmentation */
#define MSC3D_OPT_VALIDATE 2     /* ComputeOptions::validate (device audit) */
/* Whole pipeline on the loaded values.  Device results:
 *   "cp_cell" (id) "cp_index" (u8)      critical points sorted by (index, cell)
 *   "arc_src" "arc_dst" (u32) "arc_mult" (u64)   sorted by (src, dst)
 *   "labels_min" (u32, V) "labels_max" (u32, Cu)  when MSC3D_OPT_SEGMENTATION
 * stage_ms[5] (nullable) receives device milliseconds of the reference's five
 * StageTimings (gradient, critical, extrema, reachability, counting). */
int msc3d_ctx_compute(msc3d_ctx* ctx, int options, double* stage_ms);

/* The same pipeline with the results delivered to HOST memory (pinned buffers give
 * full PCIe/C2C bandwidth): every output is copied on a second stream as soon as it
 * is final, overlapping the later stages.  Capacities: cp_cell_cap / cp_index_cap in
 * bytes, arc_cap in arcs; labels_min (n_verts u32) / labels_max (n_cubes u32) only
 * with MSC3D_OPT_SEGMENTATION (NULL: not copied).  Too small a buffer ->
 * MSC3D_ERR_INVALID.  On return n_cp / n_arcs hold the sizes; the device arrays of
 * msc3d_ctx_compute stay valid as well.  Multiplicities travel as one byte per arc and
 * the (sorted) sources as one-byte steps, each plus an escape list, and are decoded
 * into arc_mult / arc_src by host threads (option "d2h_narrow"); scalar "d2h_bytes" =
 * the bytes that crossed the bus. */
typedef struct msc3d_host_outputs {
    void* cp_cell;
    uint64_t cp_cell_cap;
    uint8_t* cp_index;
    uint64_t cp_index_cap;
    uint32_t* arc_src;
    uint32_t* arc_dst;
    uint64_t* arc_mult;
    uint64_t arc_cap;
    uint32_t* labels_min;
    uint32_t* labels_max;
    uint64_t n_cp;   /* out */
    uint64_t n_arcs; /* out */
} msc3d_host_outputs;
int msc3d_ctx_compute_host(msc3d_ctx* ctx, int options, double* stage_ms, msc3d_host_outputs* out);
/* The device outputs of the last computation (msc3d_ctx_compute, or the full context of a
 * multi-GPU step) delivered to host buffers the way msc3d_ctx_compute_host delivers them
 * (narrow multiplicities / sources decoded on host threads).  Not in the reference. */
int msc3d_ctx_deliver_host(msc3d_ctx* ctx, msc3d_host_outputs* out);
/* Host samples in, host results out: msc3d_ctx_load_values + msc3d_ctx_compute_host in
 * one call, with the upload overlapped too -- the samples go up in z-chunks and the
 * gradient's tile layers start as soon as the planes they read have arrived.  Same
 * results and errors (non-finite sample -> MSC3D_ERR_INVALID). */
int msc3d_ctx_compute_host_values(msc3d_ctx* ctx, msc3d_dims dims, int value_type, const void* host_values,
                                  int options, double* stage_ms, msc3d_host_outputs* out);

/* The pipeline after the gradient, on the installed codes (msc3d_ctx_load_codes /
 * msc3d_ctx_bind_codes): extremum forests are built from the codes; the saddle
 * stages use shard `shard` of `n_shards` balanced contiguous slices of the critical
 * 1-cells as sources (crit1[c1*shard/n_shards, c1*(shard+1)/n_shards)).  With one
 * shard the results equal msc3d_ctx_compute's.  With several (a rank of a multi-GPU
 * run) the 1s->2s arcs of the shard's 1-saddles -- a contiguous block of the global
 * sorted arc list -- are left in "arcB_src", "arcB_dst" (cp ids), "arcB_mult"; the
 * min->1s and 2s->max blocks are always in "arcA_*" / "arcC_*", the critical points
 * and labels as for msc3d_ctx_compute. */
int msc3d_ctx_compute_codes(msc3d_ctx* ctx, int options, uint32_t shard, uint32_t n_shards,
                            double* stage_ms);

/* FNV-1a 64 over the widened f64 samples (msc.cpp:31-42), host-side, of the values
 * last loaded from host memory. */
uint64_t msc3d_field_hash_f64(const double* values, uint64_t n);
uint64_t msc3d_field_hash_f32(const float* values, uint64_t n);

/* ---- multi-GPU (the reference has no counterpart) ---------------------
 * One process per GPU.  A communicator is NCCL (libnccl.so.2 loaded at run time) or a
 * host transport: an allgather over host buffers supplied by the caller (e.g.
 * torch.distributed/gloo when several ranks share one GPU).  msc3d_mg_compute runs one
 * step on rank r of G (paper_2009_03707_b200/csrc/multigpu.cu): P2P halo exchange of
 * kHalo = 2 vertex planes, z-slab gradient, per-slab critical compaction (counts
 * allgather + lists allgather-v), allgather-v of the owned code planes, extrema on the
 * replicated codes, reachability + counting from the rank's 1-saddle slice,
 * allgather-v of the arc blocks.  Every rank ends with the whole complex in its
 * full-grid context (msc3d_mg_full_ctx): "cp_cell", "cp_index", "arc_src/dst/mult",
 * "labels_min/max". */
typedef struct msc3d_comm msc3d_comm;
typedef struct msc3d_mg msc3d_mg;
typedef struct msc3d_host_transport {
    void* user;
    /* every rank contributes `bytes` from send; recv receives world*bytes in rank order;
     * returns 0 on success */
    int (*allgather)(void* user, const void* send, void* recv, uint64_t bytes);
} msc3d_host_transport;

/* Slab plan of rank `rank` of `world` over nz vertex planes: out = {z0, z1 (own vertex
 * planes), lo, hi (slab grid incl. halo), own_c0, own_c1 (own lattice planes),
 * local_c0 (first own lattice plane in the slab's lattice)}.  Host-only.
 * MSC3D_ERR_INVALID if a rank would own fewer than 2 planes (the halo depth). */
int msc3d_mg_plan(int64_t nz, int world, int rank, int64_t out[7]);
int msc3d_nccl_unique_id(uint8_t out[128]);
int msc3d_comm_create_nccl(msc3d_comm** out, const uint8_t id[128], int rank, int world, int device);
int msc3d_comm_create_host(msc3d_comm** out, const msc3d_host_transport* t, int rank, int world);
void msc3d_comm_destroy(msc3d_comm* c);
int msc3d_mg_create(msc3d_mg** out, msc3d_comm* comm, int device);
void msc3d_mg_destroy(msc3d_mg* g);
msc3d_ctx* msc3d_mg_full_ctx(msc3d_mg* g);
msc3d_ctx* msc3d_mg_slab_ctx(msc3d_mg* g);
int msc3d_mg_set_stream(msc3d_mg* g, void* stream);
/* own_values: device pointer to this rank's own vertex planes [z0, z1) (x-fastest).
 * stage_ms (optional, 7 doubles): halo+slab gradient, slab critical + gathers, extrema,
 * reachability, counting, arc gather, whole step. */
int msc3d_mg_compute(msc3d_mg* g, msc3d_dims dims, int value_type, const void* own_values, int options,
                     double* stage_ms);

#ifdef __cplusplus
}
#endif
#endif /* MSC3D_CUDA_H */

// Stage orchestration (host code driving the device kernels for one context).
#pragma once

#include <cstdint>

#include "ctx.cuh"

namespace msc3d_stage {

int gradient(msc3d_ctx* ctx, bool with_forests);
int critical(msc3d_ctx* ctx);
int forest(msc3d_ctx* ctx, int dim);
int roots_sync(msc3d_ctx* ctx, int dim);
int se_arcs(msc3d_ctx* ctx);
int mark(msc3d_ctx* ctx, const void* host_sources, std::uint64_t n_sources);
int minor(msc3d_ctx* ctx);
int count(msc3d_ctx* ctx);
int count_minor(msc3d_ctx* ctx, const void* ones, std::uint64_t n1, const void* juncs,
                std::uint64_t nj, const void* twos, std::uint64_t n2,
                const std::uint32_t* const* src, const std::uint32_t* const* dst,
                const std::uint64_t* const* mult, const std::uint64_t* count, int id_width);
int compute(msc3d_ctx* ctx, int options, double* stage_ms, const msc3d_host_outputs* host = nullptr);
int deliver_host(msc3d_ctx* ctx, const msc3d_host_outputs* host);
int compute_streamed(msc3d_ctx* ctx, const void* host_values, int value_type, int options, double* stage_ms,
                     const msc3d_host_outputs* host);
// validate_gradient on the device (MSC3D_OPT_VALIDATE; audit.cu)
int validate(msc3d_ctx* ctx);
// out = {matching_violations, cells_in_closed_vpath, acyclicity_checked, degenerate}
// (GradientReport, gradient.hpp:83-91) of the context's codes; offending cells in
// array "audit_samples"
int audit_gradient(msc3d_ctx* ctx, std::uint64_t max_cells_for_cycles, std::uint64_t out[4]);
// boundary_check (msc.cpp:149-167) over device arrays; odd pairs -> "odd_top", "odd_low"
int boundary_check(msc3d_ctx* ctx, std::uint64_t n_cp, const std::uint8_t* cp_index, std::uint64_t n_arcs,
                   const std::uint32_t* src, const std::uint32_t* dst, const std::uint64_t* mult,
                   std::uint64_t* n_odd);
// sharded == false: sources crit1[a, a + b); true: shard a of b balanced slices
int compute_from_codes(msc3d_ctx* ctx, int options, double* stage_ms, const msc3d_host_outputs* host,
                       bool forests_ready, std::uint64_t a, std::uint64_t b, cudaEvent_t grad_t0,
                       bool sharded = false);
int load_marked(msc3d_ctx* ctx, const std::uint8_t* host_marked, const void* ones, std::uint64_t n1,
                const void* twos, std::uint64_t n2);
int sp_op(msc3d_ctx* ctx, int op, std::uint32_t xr, std::uint32_t xc, const std::uint64_t* xp,
          const std::uint32_t* xcol, const std::uint64_t* xcnt, std::uint32_t yr, std::uint32_t yc,
          const std::uint64_t* yp, const std::uint32_t* ycol, const std::uint64_t* ycnt);

}  // namespace msc3d_stage

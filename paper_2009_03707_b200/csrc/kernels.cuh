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
                    std::uint32_t* parent0, std::uint32_t* parent3, cudaStream_t stream);

// critical.cu
int launch_critical_count(const std::uint8_t* codes, const Dims& d, std::uint64_t* d_totals,
                          cudaStream_t s, int num_sms);
int launch_critical_compact(const std::uint8_t* codes, const Dims& d, Workspace& ws,
                            void* const outs[4], int id_width, std::uint64_t* d_totals,
                            cudaStream_t s);
int launch_saddle_count(const std::uint8_t* codes, const Dims& d, std::uint64_t* d_totals,
                        cudaStream_t s, int num_sms);
int launch_saddle_compact(const std::uint8_t* codes, const Dims& d, Workspace& ws, void* out,
                          int id_width, std::uint64_t* d_totals, cudaStream_t s);
int launch_marked_critical_count(const std::uint8_t* codes, const std::uint8_t* marked,
                                 const Dims& d, std::uint64_t* d_totals, cudaStream_t s,
                                 int num_sms);
int launch_marked_critical_compact(const std::uint8_t* codes, const std::uint8_t* marked,
                                   const Dims& d, Workspace& ws, void* const outs[4],
                                   int id_width, std::uint64_t* d_totals, cudaStream_t s);

}  // namespace msc3d_dev

namespace msc3d_dev {
// primitives.cu
int scan_u32(const std::uint32_t* in, std::uint64_t n, std::uint64_t* out, std::uint64_t* d_total,
             Workspace& ws, cudaStream_t s);

// extrema.cu
int launch_forest(const std::uint8_t* codes, const Dims& d, int dim, std::uint32_t* parent,
                  cudaStream_t s, int num_sms);
int launch_double_round(const std::uint32_t* in, std::uint32_t* out, std::uint64_t n,
                        unsigned int* changed, cudaStream_t s, int num_sms);
int launch_jump_round(std::uint32_t* p, std::uint64_t n, unsigned int* changed, cudaStream_t s,
                      int num_sms);
int launch_scatter_remap(const void* crit, std::uint64_t n, int id_width, const Dims& d, int dim,
                         std::uint32_t base, std::uint32_t* remap, cudaStream_t s, int num_sms);
int launch_gather(const std::uint32_t* label, const std::uint32_t* remap, std::uint64_t n,
                  std::uint32_t* out, cudaStream_t s, int num_sms);
int launch_se_slots(const std::uint8_t* codes, const Dims& d, const void* saddles,
                    std::uint64_t ns, int id_width, const std::uint32_t* l0,
                    const std::uint32_t* l3, std::uint64_t* slot, std::uint32_t* cnt,
                    cudaStream_t s, int num_sms);
int launch_se_write(const void* saddles, std::uint64_t ns, int id_width,
                    const std::uint64_t* slot, const std::uint64_t* off, void* out_s, void* out_e,
                    std::uint32_t* out_m, cudaStream_t s, int num_sms);
}  // namespace msc3d_dev

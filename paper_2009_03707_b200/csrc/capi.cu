// extern "C" boundary (include/msc3d_cuda.h): context management, ingestion, and
// the per-stage entry points.  No exceptions, no C++ types across the ABI.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "ctx.cuh"
#include "kernels.cuh"
#include "stages.cuh"

using msc3d_dev::Dims;

namespace msc3d_dev {
std::uint64_t& launch_counter() {
    static std::uint64_t n = 0;
    return n;
}
}  // namespace msc3d_dev

namespace {

__global__ void k_check_finite_f32(const float* v, std::uint64_t n, unsigned long long* bad) {
    for (std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<std::uint64_t>(gridDim.x) * blockDim.x)
        if (!isfinite(v[i])) atomicMin(bad, static_cast<unsigned long long>(i));
}
__global__ void k_check_finite_f64(const double* v, std::uint64_t n, unsigned long long* bad) {
    for (std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<std::uint64_t>(gridDim.x) * blockDim.x)
        if (!isfinite(v[i])) atomicMin(bad, static_cast<unsigned long long>(i));
}

int set_dims(msc3d_ctx* ctx, msc3d_dims dims) {
    const int rc = msc3d_check_dims(dims, 1);
    if (rc != MSC3D_OK) return rc;
    if (static_cast<std::uint64_t>(dims.nx) * dims.ny * dims.nz >= 0xffffffffull)
        return MSC3D_ERR_INVALID;  // dense vertex indices are u32
    const Dims nd = Dims::make(dims.nx, dims.ny, dims.nz);
    ctx->dims = nd;
    ctx->have_dims = true;
    return MSC3D_OK;
}

int validate_values(msc3d_ctx* ctx) {
    const Dims& d = ctx->dims;
    MSC3D_CUDA_TRY(cudaMemsetAsync(ctx->d_small, 0xff, 8, ctx->stream));
    const unsigned grid = static_cast<unsigned>(
        std::min<std::uint64_t>((d.n_verts + 255) / 256, 16ull * ctx->num_sms));
    auto* bad = reinterpret_cast<unsigned long long*>(ctx->d_small);
    if (ctx->value_type == MSC3D_VALUE_F64)
        k_check_finite_f64<<<grid, 256, 0, ctx->stream>>>(static_cast<const double*>(ctx->values),
                                                          d.n_verts, bad);
    else
        k_check_finite_f32<<<grid, 256, 0, ctx->stream>>>(static_cast<const float*>(ctx->values),
                                                          d.n_verts, bad);
    msc3d_dev::count_launch();
    MSC3D_CUDA_TRY(cudaGetLastError());
    const int rc = ctx->fetch_small(1);
    if (rc != MSC3D_OK) return rc;
    if (ctx->h_small[0] != ~0ull) return MSC3D_ERR_INVALID;
    return MSC3D_OK;
}

}  // namespace

extern "C" {

const char* msc3d_status_string(int status) {
    switch (status) {
        case MSC3D_OK: return "ok";
        case MSC3D_ERR_INVALID: return "invalid_argument";
        case MSC3D_ERR_OVERFLOW: return "overflow_error: path count exceeds 64 bits";
        case MSC3D_ERR_RUNTIME: return "runtime_error";
        case MSC3D_ERR_CUDA: return "cuda error";
        case MSC3D_ERR_NOMEM: return "device out of memory";
        case MSC3D_ERR_IO: return "i/o error";
        case MSC3D_ERR_STATE: return "stage inputs missing";
        default: return "unknown status";
    }
}

int msc3d_check_dims(msc3d_dims d, int allow_wide) {
    if (d.nx < 2 || d.ny < 2 || d.nz < 2) return MSC3D_ERR_INVALID;
    if (d.nx > (1ll << 31) || d.ny > (1ll << 31) || d.nz > (1ll << 31)) return MSC3D_ERR_INVALID;
    if (!allow_wide && msc3d_total_cells(d) > 0xffffffffull) return MSC3D_ERR_INVALID;
    return MSC3D_OK;
}

std::uint64_t msc3d_total_cells(msc3d_dims d) {
    return static_cast<std::uint64_t>(2 * d.nx - 1) * static_cast<std::uint64_t>(2 * d.ny - 1) *
           static_cast<std::uint64_t>(2 * d.nz - 1);
}

int msc3d_id_width(msc3d_dims d) { return msc3d_total_cells(d) <= 0xffffffffull ? 4 : 8; }

int msc3d_ctx_create(msc3d_ctx** out, int device) {
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        cudaGetLastError();
        return MSC3D_ERR_CUDA;
    }
    if (device < 0 || device >= n) return MSC3D_ERR_INVALID;
    MSC3D_CUDA_TRY(cudaSetDevice(device));
    auto* ctx = new msc3d_ctx();
    ctx->device = device;
    cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device);
    if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaMalloc(&ctx->d_small, msc3d_ctx::kSmall * 8) != cudaSuccess ||
        cudaHostAlloc(&ctx->h_small, msc3d_ctx::kSmall * 8, cudaHostAllocMapped) != cudaSuccess ||
        cudaHostGetDevicePointer(reinterpret_cast<void**>(&ctx->h_small_dev), ctx->h_small, 0) != cudaSuccess) {
        delete ctx;
        return MSC3D_ERR_CUDA;
    }
    ctx->own_stream = true;
    ctx->launches_at_create = msc3d_dev::launch_counter();
    *out = ctx;
    return MSC3D_OK;
}

void msc3d_ctx_destroy(msc3d_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    delete ctx;
}

int msc3d_ctx_set_stream(msc3d_ctx* ctx, void* stream) {
    if (!stream) return MSC3D_OK;
    if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
    ctx->stream = static_cast<cudaStream_t>(stream);
    ctx->own_stream = false;
    return MSC3D_OK;
}

void* msc3d_ctx_stream(msc3d_ctx* ctx) { return ctx->stream; }

int msc3d_ctx_sync(msc3d_ctx* ctx) {
    MSC3D_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    return MSC3D_OK;
}

std::uint64_t msc3d_ctx_launches(msc3d_ctx* ctx) {
    return msc3d_dev::launch_counter() - ctx->launches_at_create;
}

int msc3d_ctx_array(msc3d_ctx* ctx, const char* name, void** device_ptr, std::uint64_t* count,
                    int* elem_bytes) {
    DevArray* a = ctx->find(name);
    if (!a) return MSC3D_ERR_STATE;
    if (device_ptr) *device_ptr = a->ptr;
    if (count) *count = a->count;
    if (elem_bytes) *elem_bytes = a->elem;
    return MSC3D_OK;
}

int msc3d_host_alloc(void** out, std::uint64_t bytes) {
    if (!out) return MSC3D_ERR_INVALID;
    *out = nullptr;
    if (cudaHostAlloc(out, bytes ? bytes : 1, cudaHostAllocDefault) != cudaSuccess) {
        cudaGetLastError();
        *out = nullptr;
        return MSC3D_ERR_NOMEM;
    }
    return MSC3D_OK;
}

void msc3d_host_free(void* p) {
    if (p) cudaFreeHost(p);
}

int msc3d_ctx_download(msc3d_ctx* ctx, const char* name, void* host, std::uint64_t capacity) {
    DevArray* a = ctx->find(name);
    if (!a) return MSC3D_ERR_STATE;
    const std::uint64_t bytes = a->count * static_cast<std::uint64_t>(a->elem);
    if (bytes > capacity) return MSC3D_ERR_INVALID;
    if (bytes)
        MSC3D_CUDA_TRY(cudaMemcpyAsync(host, a->ptr, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    MSC3D_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    return MSC3D_OK;
}

int msc3d_ctx_cp_values(msc3d_ctx* ctx) {
    if (!ctx) return MSC3D_ERR_INVALID;
    DevArray* cells = ctx->find("cp_cell");
    if (!cells || !ctx->values) return MSC3D_ERR_STATE;
    auto* out = static_cast<double*>(ctx->ensure("cp_value", std::max<std::uint64_t>(1, cells->count), 8));
    if (!out) return MSC3D_ERR_NOMEM;
    ctx->find("cp_value")->count = cells->count;
    return msc3d_dev::launch_cp_values(ctx->find("cp_cell")->ptr, ctx->find("cp_cell")->elem, cells->count, ctx->dims,
                                       ctx->values, ctx->value_type, out, ctx->stream, ctx->num_sms);
}

int msc3d_ctx_set_option(msc3d_ctx* ctx, const char* name, std::int64_t value) {
    if (!ctx || !name) return MSC3D_ERR_INVALID;
    const std::string n(name);
    if (n == "wide_ids") {
        ctx->force_wide = value != 0;
    } else if (n == "kahn_switch_below") {
        if (value < 1) return MSC3D_ERR_INVALID;
        ctx->kahn_switch_below = static_cast<std::uint64_t>(value);
    } else if (n == "exact_batch_rows") {  // rows per batch of the exact A* check (0 = by memory)
        if (value < 0) return MSC3D_ERR_INVALID;
        ctx->exact_batch_rows = static_cast<std::uint64_t>(value);
    } else if (n == "frontier_cap") {  // initial BFS frontier entries (0 = 4 x sources)
        if (value < 0) return MSC3D_ERR_INVALID;
        ctx->frontier_cap = static_cast<std::uint64_t>(value);
    } else if (n == "side_stream") {  // extremum-side assembly beside the saddle stages
        ctx->side_assembly = value != 0;
    } else if (n == "kahn_async") {  // Kahn's tail without rounds (k_count_async)
        ctx->kahn_async = value != 0;
    } else if (n == "d2h_narrow") {  // multiplicities cross the bus as bytes + escapes (default 1)
        ctx->d2h_narrow = value != 0;
    } else if (n == "d2h_escape_cap") {  // escape-list entries per arc block (0 = n / 16 + 1024)
        if (value < 0) return MSC3D_ERR_INVALID;
        ctx->d2h_escape_cap = static_cast<std::uint64_t>(value);
    } else if (n == "d2h_narrow_max") {  // largest multiplicity sent as a byte (<= 254)
        if (value < 0 || value > 254) return MSC3D_ERR_INVALID;
        ctx->d2h_narrow_max = static_cast<std::uint64_t>(value);
    } else if (n == "release_transients") {  // 1: free stage scratch early on any grid; 0: never; -1: auto
        ctx->force_release = value > 0;
        ctx->never_release = value == 0;
    } else if (n == "term_rank_words") {  // the large-grid 2-saddle rank lookup on any grid
        ctx->term_rank_words = value != 0;
    } else {
        return MSC3D_ERR_INVALID;
    }
    return MSC3D_OK;
}

int msc3d_ctx_scalar(msc3d_ctx* ctx, const char* name, std::int64_t* value) {
    if (!ctx || !name || !value) return MSC3D_ERR_INVALID;
    if (!std::strcmp(name, "device_bytes_held")) {
        *value = static_cast<std::int64_t>(ctx->held_bytes());
        return MSC3D_OK;
    }
    if (!std::strcmp(name, "device_bytes_peak")) {
        *value = static_cast<std::int64_t>(ctx->peak_held);
        return MSC3D_OK;
    }
    if (!std::strcmp(name, "host_syncs")) {  // host round trips since the context was created
        *value = static_cast<std::int64_t>(ctx->n_fetch);
        return MSC3D_OK;
    }
    if (!std::strcmp(name, "host_sync_us")) {  // host time spent waiting in them
        *value = static_cast<std::int64_t>(ctx->fetch_us);
        return MSC3D_OK;
    }
    auto it = ctx->scalars.find(name);
    if (it == ctx->scalars.end()) return MSC3D_ERR_STATE;
    *value = it->second;
    return MSC3D_OK;
}

int msc3d_ctx_load_values(msc3d_ctx* ctx, msc3d_dims dims, int value_type, const void* host) {
    int rc = set_dims(ctx, dims);
    if (rc != MSC3D_OK) return rc;
    if (value_type != MSC3D_VALUE_F32 && value_type != MSC3D_VALUE_F64) return MSC3D_ERR_INVALID;
    const int elem = value_type == MSC3D_VALUE_F64 ? 8 : 4;
    void* p = ctx->ensure("values", ctx->dims.n_verts, elem);
    if (!p) return MSC3D_ERR_NOMEM;
    MSC3D_CUDA_TRY(cudaMemcpyAsync(p, host, ctx->dims.n_verts * elem, cudaMemcpyHostToDevice,
                                   ctx->stream));
    ctx->value_type = value_type;
    ctx->values = p;
    return validate_values(ctx);
}

// read_volume (volume.cpp:67-96): size check -> invalid_argument, unreadable ->
// IoError, either endianness, widening.  u8/u16/f32 samples are exactly
// representable in f32, so the device keeps them as f32; f64 stays
// f64.  Non-finite samples are rejected on the device.
int msc3d_ctx_read_volume(msc3d_ctx* ctx, const char* path, msc3d_dims dims, const char* dtype,
                          int big_endian) {
    int rc = msc3d_check_dims(dims, 1);
    if (rc != MSC3D_OK) return rc;
    int width = 0;
    const std::string t = dtype ? dtype : "";
    if (t == "u8") width = 1;
    else if (t == "u16") width = 2;
    else if (t == "f32") width = 4;
    else if (t == "f64") width = 8;
    else return MSC3D_ERR_INVALID;
    std::FILE* fp = std::fopen(path, "rb");
    if (!fp) return MSC3D_ERR_IO;
    std::fseek(fp, 0, SEEK_END);
    const long long size = std::ftell(fp);
    std::fseek(fp, 0, SEEK_SET);
    const std::uint64_t nv = static_cast<std::uint64_t>(dims.nx) * dims.ny * dims.nz;
    if (size < 0 || static_cast<std::uint64_t>(size) != nv * width) {
        std::fclose(fp);
        return MSC3D_ERR_INVALID;
    }
    std::vector<unsigned char> raw(static_cast<std::size_t>(size));
    const std::size_t got = raw.empty() ? 0 : std::fread(raw.data(), 1, raw.size(), fp);
    std::fclose(fp);
    if (got != raw.size()) return MSC3D_ERR_IO;
    auto load = [&](std::size_t i) {
        std::uint64_t v = 0;
        for (int k = 0; k < width; ++k) {
            const int byte = big_endian ? width - 1 - k : k;
            v |= static_cast<std::uint64_t>(raw[i * width + byte]) << (8 * k);
        }
        return v;
    };
    if (width == 8) {
        std::vector<double> v(nv);
        for (std::uint64_t i = 0; i < nv; ++i) {
            const std::uint64_t b = load(i);
            std::memcpy(&v[i], &b, 8);
        }
        return msc3d_ctx_load_values(ctx, dims, MSC3D_VALUE_F64, v.data());
    }
    std::vector<float> v(nv);
    for (std::uint64_t i = 0; i < nv; ++i) {
        const std::uint64_t b = load(i);
        if (width == 4) {
            const std::uint32_t b32 = static_cast<std::uint32_t>(b);
            std::memcpy(&v[i], &b32, 4);
        } else {
            v[i] = static_cast<float>(b);
        }
    }
    return msc3d_ctx_load_values(ctx, dims, MSC3D_VALUE_F32, v.data());
}

int msc3d_ctx_bind_values(msc3d_ctx* ctx, msc3d_dims dims, int value_type, const void* dev) {
    int rc = set_dims(ctx, dims);
    if (rc != MSC3D_OK) return rc;
    if (value_type != MSC3D_VALUE_F32 && value_type != MSC3D_VALUE_F64) return MSC3D_ERR_INVALID;
    ctx->value_type = value_type;
    ctx->values = dev;
    return MSC3D_OK;
}

int msc3d_ctx_gradient(msc3d_ctx* ctx) {
    if (!ctx->values) return MSC3D_ERR_STATE;
    return msc3d_stage::gradient(ctx, /*with_forests=*/false);
}

int msc3d_ctx_load_codes(msc3d_ctx* ctx, msc3d_dims dims, const std::uint8_t* host_codes) {
    int rc = set_dims(ctx, dims);
    if (rc != MSC3D_OK) return rc;
    void* p = ctx->ensure("codes", ctx->dims.n_cells, 1);
    if (!p) return MSC3D_ERR_NOMEM;
    MSC3D_CUDA_TRY(cudaMemcpyAsync(p, host_codes, ctx->dims.n_cells, cudaMemcpyHostToDevice,
                                   ctx->stream));
    ctx->crit_counts_valid = false;
    return MSC3D_OK;
}

int msc3d_ctx_critical(msc3d_ctx* ctx) {
    if (!ctx->find("codes")) return MSC3D_ERR_STATE;
    return msc3d_stage::critical(ctx);
}

int msc3d_ctx_forest(msc3d_ctx* ctx, int dim) {
    if (dim != 0 && dim != 3) return MSC3D_ERR_INVALID;
    if (!ctx->find("codes")) return MSC3D_ERR_STATE;
    return msc3d_stage::forest(ctx, dim);
}

int msc3d_ctx_load_parent(msc3d_ctx* ctx, int dim, const std::uint32_t* host_parent,
                          std::uint64_t n) {
    if (dim != 0 && dim != 3) return MSC3D_ERR_INVALID;
    const std::string name = dim == 0 ? "parent0" : "parent3";
    void* p = ctx->ensure(name, n, 4);
    if (!p) return MSC3D_ERR_NOMEM;
    if (n) MSC3D_CUDA_TRY(cudaMemcpyAsync(p, host_parent, n * 4, cudaMemcpyHostToDevice, ctx->stream));
    return MSC3D_OK;
}

int msc3d_ctx_roots(msc3d_ctx* ctx, int dim) {
    if (dim != 0 && dim != 3) return MSC3D_ERR_INVALID;
    if (!ctx->find(dim == 0 ? "parent0" : "parent3")) return MSC3D_ERR_STATE;
    return msc3d_stage::roots_sync(ctx, dim);
}

int msc3d_ctx_load_labels(msc3d_ctx* ctx, const std::uint32_t* l0, const std::uint32_t* l3) {
    if (!ctx->have_dims) return MSC3D_ERR_STATE;
    void* a = ctx->ensure("label0", ctx->dims.n_verts, 4);
    void* b = ctx->ensure("label3", ctx->dims.n_cubes, 4);
    if (!a || !b) return MSC3D_ERR_NOMEM;
    MSC3D_CUDA_TRY(cudaMemcpyAsync(a, l0, ctx->dims.n_verts * 4, cudaMemcpyHostToDevice, ctx->stream));
    if (ctx->dims.n_cubes)
        MSC3D_CUDA_TRY(cudaMemcpyAsync(b, l3, ctx->dims.n_cubes * 4, cudaMemcpyHostToDevice, ctx->stream));
    return MSC3D_OK;
}

int msc3d_ctx_se_arcs(msc3d_ctx* ctx) {
    if (!ctx->find("codes") || !ctx->find("label0") || !ctx->find("label3")) return MSC3D_ERR_STATE;
    return msc3d_stage::se_arcs(ctx);
}

int msc3d_ctx_mark(msc3d_ctx* ctx, const void* host_sources, std::uint64_t n_sources) {
    if (!ctx->find("codes")) return MSC3D_ERR_STATE;
    return msc3d_stage::mark(ctx, host_sources, n_sources);
}

int msc3d_ctx_load_marked(msc3d_ctx* ctx, const std::uint8_t* host_marked, const void* ones,
                          std::uint64_t n1, const void* twos, std::uint64_t n2) {
    return msc3d_stage::load_marked(ctx, host_marked, ones, n1, twos, n2);
}

int msc3d_sp_op(msc3d_ctx* ctx, int op, std::uint32_t xr, std::uint32_t xc, const std::uint64_t* xp,
                const std::uint32_t* xcol, const std::uint64_t* xcnt, std::uint32_t yr, std::uint32_t yc,
                const std::uint64_t* yp, const std::uint32_t* ycol, const std::uint64_t* ycnt) {
    if (op != 0 && op != 1) return MSC3D_ERR_INVALID;
    return msc3d_stage::sp_op(ctx, op, xr, xc, xp, xcol, xcnt, yr, yc, yp, ycol, ycnt);
}

int msc3d_ctx_validate_gradient(msc3d_ctx* ctx, std::uint64_t max_cells_for_cycles, std::uint64_t out[4]) {
    if (!ctx || !out) return MSC3D_ERR_INVALID;
    return msc3d_stage::audit_gradient(ctx, max_cells_for_cycles, out);
}

int msc3d_ctx_boundary_check(msc3d_ctx* ctx, std::uint64_t* n_odd) {
    if (!ctx || !n_odd) return MSC3D_ERR_INVALID;
    DevArray* idx = ctx->find("cp_index");
    DevArray* src = ctx->find("arc_src");
    DevArray* dst = ctx->find("arc_dst");
    DevArray* mul = ctx->find("arc_mult");
    if (!idx || !src || !dst || !mul) return MSC3D_ERR_STATE;
    return msc3d_stage::boundary_check(ctx, idx->count, static_cast<const std::uint8_t*>(idx->ptr), src->count,
                                       static_cast<const std::uint32_t*>(src->ptr),
                                       static_cast<const std::uint32_t*>(dst->ptr),
                                       static_cast<const std::uint64_t*>(mul->ptr), n_odd);
}

int msc3d_boundary_check_host(msc3d_ctx* ctx, std::uint64_t n_cp, const std::uint8_t* cp_index, std::uint64_t n_arcs,
                              const std::uint32_t* src, const std::uint32_t* dst, const std::uint64_t* mult,
                              std::uint64_t* n_odd) {
    if (!ctx || !n_odd) return MSC3D_ERR_INVALID;
    for (std::uint64_t i = 0; i < n_arcs; ++i)
        if (src[i] >= n_cp || dst[i] >= n_cp) return MSC3D_ERR_INVALID;
    auto* di = static_cast<std::uint8_t*>(ctx->ensure("bc_cp_index", std::max<std::uint64_t>(n_cp, 1), 1));
    auto* ds = static_cast<std::uint32_t*>(ctx->ensure("bc_src", std::max<std::uint64_t>(n_arcs, 1), 4));
    auto* dd = static_cast<std::uint32_t*>(ctx->ensure("bc_dst", std::max<std::uint64_t>(n_arcs, 1), 4));
    auto* dm = static_cast<std::uint64_t*>(ctx->ensure("bc_mult", std::max<std::uint64_t>(n_arcs, 1), 8));
    if (!di || !ds || !dd || !dm) return MSC3D_ERR_NOMEM;
    if (n_cp) MSC3D_CUDA_TRY(cudaMemcpyAsync(di, cp_index, n_cp, cudaMemcpyHostToDevice, ctx->stream));
    if (n_arcs) {
        MSC3D_CUDA_TRY(cudaMemcpyAsync(ds, src, n_arcs * 4, cudaMemcpyHostToDevice, ctx->stream));
        MSC3D_CUDA_TRY(cudaMemcpyAsync(dd, dst, n_arcs * 4, cudaMemcpyHostToDevice, ctx->stream));
        MSC3D_CUDA_TRY(cudaMemcpyAsync(dm, mult, n_arcs * 8, cudaMemcpyHostToDevice, ctx->stream));
    }
    return msc3d_stage::boundary_check(ctx, n_cp, di, n_arcs, ds, dd, dm, n_odd);
}

int msc3d_ctx_minor(msc3d_ctx* ctx) {
    if (!ctx->find("marked")) return MSC3D_ERR_STATE;
    return msc3d_stage::minor(ctx);
}

int msc3d_ctx_count(msc3d_ctx* ctx) {
    if (!ctx->find("marked")) return MSC3D_ERR_STATE;
    return msc3d_stage::count(ctx);
}

int msc3d_ctx_count_minor(msc3d_ctx* ctx, const void* ones, std::uint64_t n1, const void* juncs,
                          std::uint64_t nj, const void* twos, std::uint64_t n2,
                          const std::uint32_t* const* src, const std::uint32_t* const* dst,
                          const std::uint64_t* const* mult, const std::uint64_t* count,
                          int id_width) {
    return msc3d_stage::count_minor(ctx, ones, n1, juncs, nj, twos, n2, src, dst, mult, count,
                                    id_width);
}

int msc3d_ctx_bind_codes(msc3d_ctx* ctx, msc3d_dims dims, const std::uint8_t* device_codes) {
    int rc = set_dims(ctx, dims);
    if (rc != MSC3D_OK) return rc;
    void* p = ctx->ensure("codes", ctx->dims.n_cells, 1);
    if (!p) return MSC3D_ERR_NOMEM;
    MSC3D_CUDA_TRY(cudaMemcpyAsync(p, device_codes, ctx->dims.n_cells, cudaMemcpyDeviceToDevice, ctx->stream));
    ctx->crit_counts_valid = false;
    return MSC3D_OK;
}

int msc3d_ctx_compute_codes(msc3d_ctx* ctx, int options, std::uint32_t shard, std::uint32_t n_shards,
                            double* stage_ms) {
    if (!ctx || n_shards == 0 || shard >= n_shards) return MSC3D_ERR_INVALID;
    if (!ctx->have_dims || !ctx->find("codes")) return MSC3D_ERR_STATE;
    ctx->crit_counts_valid = false;
    if (options & MSC3D_OPT_VALIDATE) {
        const int rc = msc3d_stage::validate(ctx);
        if (rc != MSC3D_OK) return rc;
    }
    const int rc = msc3d_stage::compute_from_codes(ctx, options, stage_ms, nullptr, false, shard, n_shards, nullptr,
                                                   /*sharded=*/true);
    if (std::getenv("MSC3D_ALLOC_TRACE")) ctx->dump_arrays("after compute_codes");
    return rc;
}

int msc3d_ctx_compute_host_values(msc3d_ctx* ctx, msc3d_dims dims, int value_type, const void* host_values,
                                  int options, double* stage_ms, msc3d_host_outputs* out) {
    if (!ctx || !out || !host_values) return MSC3D_ERR_INVALID;
    if (value_type != MSC3D_VALUE_F32 && value_type != MSC3D_VALUE_F64) return MSC3D_ERR_INVALID;
    const int rc = set_dims(ctx, dims);
    if (rc != MSC3D_OK) return rc;
    return msc3d_stage::compute_streamed(ctx, host_values, value_type, options, stage_ms, out);
}

int msc3d_ctx_deliver_host(msc3d_ctx* ctx, msc3d_host_outputs* out) {
    if (!ctx || !out) return MSC3D_ERR_INVALID;
    return msc3d_stage::deliver_host(ctx, out);
}

int msc3d_ctx_compute_host(msc3d_ctx* ctx, int options, double* stage_ms, msc3d_host_outputs* out) {
    if (!ctx || !out) return MSC3D_ERR_INVALID;
    if (!ctx->values) return MSC3D_ERR_STATE;
    return msc3d_stage::compute(ctx, options, stage_ms, out);
}

int msc3d_ctx_compute(msc3d_ctx* ctx, int options, double* stage_ms) {
    if (!ctx->values) return MSC3D_ERR_STATE;
    return msc3d_stage::compute(ctx, options, stage_ms);
}

std::uint64_t msc3d_field_hash_f64(const double* values, std::uint64_t n) {
    // FNV-1a 64 over the little-endian bytes of each double (msc.cpp:31-42).
    std::uint64_t h = 0xcbf29ce484222325ull;
    for (std::uint64_t i = 0; i < n; ++i) {
        std::uint64_t bits;
        std::memcpy(&bits, &values[i], 8);
        for (int b = 0; b < 64; b += 8) {
            h ^= (bits >> b) & 0xffu;
            h *= 0x100000001b3ull;
        }
    }
    return h;
}

std::uint64_t msc3d_field_hash_f32(const float* values, std::uint64_t n) {
    std::uint64_t h = 0xcbf29ce484222325ull;
    for (std::uint64_t i = 0; i < n; ++i) {
        const double w = static_cast<double>(values[i]);  // the reference widens first
        std::uint64_t bits;
        std::memcpy(&bits, &w, 8);
        for (int b = 0; b < 64; b += 8) {
            h ^= (bits >> b) & 0xffu;
            h *= 0x100000001b3ull;
        }
    }
    return h;
}

}  // extern "C"

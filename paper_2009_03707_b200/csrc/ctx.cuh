// The context behind msc3d_ctx: device, stream, named device arrays, scalars and
// scratch.  Arrays keep their capacity across calls so a repeated pipeline run on
// the same grid allocates nothing.
#pragma once

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <string>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"

struct DevArray {
    void* ptr = nullptr;
    std::uint64_t count = 0;
    int elem = 1;
    std::size_t cap = 0;
};

struct msc3d_ctx {
    int device = 0;
    int num_sms = 148;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    msc3d_dev::Dims dims{};
    bool have_dims = false;
    bool crit_counts_valid = false;  // d_small[40..43] hold the codes' critical counts
    bool crit_external = false;      // crit0..3 + scalars c0..c3 installed by the caller (multigpu.cu)
    int value_type = MSC3D_VALUE_F32;
    // msc3d_ctx_set_option: "wide_ids" forces 64-bit cell-id lists on any grid (the
    // path configs 4-5 take, testable on small grids); "kahn_switch_below" is the
    // frontier size at which the counting kernel hands over to its tail configuration.
    bool force_wide = false;
    std::uint64_t kahn_switch_below = 1ull << 18;
    bool kahn_async = true;  // "kahn_async": Kahn's tail without rounds (k_count_async); 0: rounds
    std::uint64_t exact_batch_rows = 0;  // "exact_batch_rows": batch of the exact A* overflow check
    std::uint64_t frontier_cap = 0;      // "frontier_cap": initial BFS frontier entries (0 = 4 x sources)
    bool term_rank_words = false;        // "term_rank_words": 2-saddle rank words on any grid
    const void* values = nullptr;  // device pointer (owned "values" array or bound)
    std::map<std::string, DevArray> arrays;
    std::map<std::string, std::int64_t> scalars;
    msc3d_dev::Workspace ws, ws2;
    static constexpr int kSmall = 256;
    std::uint64_t* d_small = nullptr;      // kSmall u64 of device scratch for totals / flags
    std::uint64_t* h_small = nullptr;      // mapped pinned mirror
    std::uint64_t* h_small_dev = nullptr;  // its device address
    std::uint64_t launches_at_create = 0;
    cudaStream_t copy = nullptr;  // device-to-host copies overlapping the pipeline
    cudaStream_t h2d = nullptr;   // host-to-device input chunks overlapping the gradient
    // host deliveries (msc3d_ctx_compute_host*): multiplicities cross the bus as one
    // byte each (+ an escape list) and are widened on host threads; "d2h_narrow" 0
    // copies the u64 arrays instead, "d2h_escape_cap" bounds the escape list (tests)
    bool d2h_narrow = true;
    std::uint64_t d2h_escape_cap = 0;
    std::uint64_t d2h_narrow_max = 254;  // largest multiplicity sent as its byte (tests: lower)
    std::map<std::string, std::pair<void*, std::size_t>> pinned;  // pinned host staging
    std::map<std::string, std::uint64_t> d2h_esc_memo;  // escape counts of the last delivery per block

    // Pinned host staging `name` of >= bytes (kept across calls), nullptr on failure.
    void* host_buf(const std::string& name, std::size_t bytes) {
        auto& b = pinned[name];
        if (b.second < bytes || !b.first) {
            if (b.first) cudaFreeHost(b.first);
            b = {nullptr, 0};
            if (cudaHostAlloc(&b.first, bytes ? bytes : 16, cudaHostAllocDefault) != cudaSuccess) {
                cudaGetLastError();
                b.first = nullptr;
                return nullptr;
            }
            b.second = bytes;
        }
        return b.first;
    }

    cudaStream_t copy_stream() {
        if (!copy && cudaStreamCreateWithFlags(&copy, cudaStreamNonBlocking) != cudaSuccess) copy = nullptr;
        return copy;
    }
    cudaStream_t side = nullptr;  // assembly kernels beside the saddle stages ("side_stream")
    bool side_assembly = false;
    cudaStream_t side_stream() {
        if (!side && cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking) != cudaSuccess) side = nullptr;
        return side;
    }
    cudaStream_t h2d_stream() {
        if (!h2d && cudaStreamCreateWithFlags(&h2d, cudaStreamNonBlocking) != cudaSuccess) h2d = nullptr;
        return h2d;
    }

    ~msc3d_ctx() {
        for (auto& kv : arrays)
            if (kv.second.ptr) cudaFree(kv.second.ptr);
        for (auto& kv : pinned)
            if (kv.second.first) cudaFreeHost(kv.second.first);
        if (d_small) cudaFree(d_small);
        if (h_small) cudaFreeHost(h_small);
        if (own_stream && stream) cudaStreamDestroy(stream);
        if (copy) cudaStreamDestroy(copy);
        if (h2d) cudaStreamDestroy(h2d);
        if (side) cudaStreamDestroy(side);
    }

    // Ensure array `name` holds `count` elements of `elem` bytes; contents undefined.
    void* ensure(const std::string& name, std::uint64_t count, int elem) {
        DevArray& a = arrays[name];
        const std::size_t bytes = static_cast<std::size_t>(count) * elem;
        if (a.cap < bytes || !a.ptr) {
            if (a.ptr) cudaFree(a.ptr);
            a.ptr = nullptr;
            a.cap = 0;
            const std::size_t want = bytes ? bytes : 16;
            if (cudaMalloc(&a.ptr, want) != cudaSuccess) {
                cudaGetLastError();
                a.ptr = nullptr;
                if (std::getenv("MSC3D_ALLOC_TRACE")) {  // development: what holds the device memory
                    std::fprintf(stderr, "msc3d: cannot allocate %s (%.2f GB)\n", name.c_str(), want / 1e9);
                    dump_arrays("at the failure");
                }
                return nullptr;
            }
            a.cap = want;
            const std::size_t held = held_bytes();
            if (held > peak_held) peak_held = held;
        }
        a.count = count;
        a.elem = elem;
        return a.ptr;
    }
    std::size_t peak_held = 0;  // high-water mark of the named arrays (bytes)
    std::size_t held_bytes() const {
        std::size_t held = 0;
        for (const auto& kv : arrays) held += kv.second.cap;
        return held;
    }
    // development (MSC3D_ALLOC_TRACE): the arrays above 256 MB that hold device memory
    void dump_arrays(const char* when) const {
        std::fprintf(stderr, "msc3d: the context holds %.2f GB %s:\n", held_bytes() / 1e9, when);
        for (const auto& kv : arrays)
            if (kv.second.cap > (std::size_t(1) << 28))
                std::fprintf(stderr, "  %-20s %8.2f GB\n", kv.first.c_str(), kv.second.cap / 1e9);
    }
    // ensure() that keeps the first `keep` bytes when it has to grow (a new buffer, the
    // bytes copied on `s`, the old one freed after the device is idle -- rare: capacities
    // persist across calls).
    void* ensure_keep(const std::string& name, std::uint64_t count, int elem, std::size_t keep, cudaStream_t s) {
        DevArray& a = arrays[name];
        const std::size_t bytes = static_cast<std::size_t>(count) * elem;
        if (a.ptr && a.cap >= bytes) {
            a.count = count;
            a.elem = elem;
            return a.ptr;
        }
        void* fresh = nullptr;
        if (cudaMalloc(&fresh, bytes ? bytes : 16) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        if (a.ptr && keep) {
            if (cudaMemcpyAsync(fresh, a.ptr, std::min(keep, a.cap), cudaMemcpyDeviceToDevice, s) != cudaSuccess ||
                cudaDeviceSynchronize() != cudaSuccess)
                return nullptr;
        } else if (a.ptr) {
            cudaDeviceSynchronize();
        }
        if (a.ptr) cudaFree(a.ptr);
        a.ptr = fresh;
        a.cap = bytes ? bytes : 16;
        a.count = count;
        a.elem = elem;
        const std::size_t held = held_bytes();
        if (held > peak_held) peak_held = held;
        return a.ptr;
    }
    DevArray* find(const std::string& name) {
        auto it = arrays.find(name);
        return it == arrays.end() ? nullptr : &it->second;
    }
    template <typename T>
    T* ptr(const std::string& name) {
        DevArray* a = find(name);
        return a ? static_cast<T*>(a->ptr) : nullptr;
    }
    std::uint64_t count(const std::string& name) {
        DevArray* a = find(name);
        return a ? a->count : 0;
    }
    void drop(const std::string& name) {
        auto it = arrays.find(name);
        if (it != arrays.end()) it->second.count = 0;
    }
    // Large grids (configs 4-5, > 2^32 cells) hand the memory of a stage's transient
    // arrays back once the stage is done (later stages allocate into it);
    // smaller grids keep them so that repeated computes allocate nothing.
    // Free stage scratch as soon as it is dead: grids above 2^32 cells (configs 4-5),
    // or any grid with the "release_transients" option (tests)
    bool force_release = false;
    bool never_release = false;
    bool release_auto = false;  // decided per compute() once the saddle counts are known
    bool release_transients() const { return force_release || (!never_release && release_auto); }
    // Above 2^32 cells the stage scratch is freed early when the saddle stages may not
    // fit beside it: their arrays grow with the saddle count (< 1 KB per saddle at every
    // measured size).  Smooth large grids (config 4: a few thousand saddles) keep
    // everything -- freeing and re-allocating costs ~19 ms per call there and does not
    // lower the peak.
    void decide_release(std::uint64_t saddles) {
        release_auto = false;
        if (dims.n_cells <= 0xffffffffull) return;
        std::size_t fr = 0, tot = 0;
        if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) {
            release_auto = true;
            return;
        }
        release_auto = saddles * 1024ull > fr;
    }
    void release(const std::string& name) {
        auto it = arrays.find(name);
        if (it == arrays.end()) return;
        if (it->second.ptr) cudaFree(it->second.ptr);  // (synchronises: large grids only)
        arrays.erase(it);
    }
    int id_width() const { return (!force_wide && dims.n_cells <= 0xffffffffull) ? 4 : 8; }
    // Copy the first n u64 of d_small to h_small and wait.  The copy is a tiny
    // kernel writing the mapped host mirror over the bus, not a DMA: a DMA would
    // queue behind bulk device-to-host output copies on the copy engine.
    int fetch_small(int n) { return fetch_range(0, n); }
    std::uint64_t n_fetch = 0;  // host round trips (development counters: scalars "host_syncs", "host_sync_us")
    double fetch_us = 0;
    int fetch_range(int first, int n) {
        if (msc3d_dev::launch_small_copy(d_small + first, h_small_dev + first, n, stream) != MSC3D_OK)
            return MSC3D_ERR_CUDA;
        const auto t0 = std::chrono::steady_clock::now();
        if (cudaStreamSynchronize(stream) != cudaSuccess) return MSC3D_ERR_CUDA;
        ++n_fetch;
        fetch_us += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
        return MSC3D_OK;
    }
};

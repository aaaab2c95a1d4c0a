// Development probe: host memory bandwidth of widening decodes on the GPU box's cores
// (u8 -> u64 multiplicities, u8 deltas -> u32 sources), into first-touch and pre-faulted
// output buffers, T threads.
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>
#include <sys/mman.h>
#include <cuda_runtime.h>
static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
int main(int argc, char** argv) {
    const std::size_t n = argc > 1 ? std::atoll(argv[1]) : 285732712;
    const int T = argc > 2 ? std::atoi(argv[2]) : std::thread::hardware_concurrency();
    std::vector<std::uint8_t> m8(n), d8(n);
    for (std::size_t i = 0; i < n; ++i) { m8[i] = (i * 2654435761u >> 13) & 3; d8[i] = (i % 3) == 0; }
    const bool pinned = argc > 3 && std::atoi(argv[3]);
    std::uint64_t* out64;
    std::uint32_t* out32;
    if (pinned) {
        cudaHostAlloc(reinterpret_cast<void**>(&out64), n * 8, cudaHostAllocDefault);
        cudaHostAlloc(reinterpret_cast<void**>(&out32), n * 4, cudaHostAllocDefault);
    } else {
        out64 = static_cast<std::uint64_t*>(std::malloc(n * 8));
        out32 = static_cast<std::uint32_t*>(std::malloc(n * 4));
    }
    std::printf("output %s\n", pinned ? "cudaHostAlloc (pinned)" : "malloc");
    for (int rep = 0; rep < 3; ++rep) {
        double t0 = now();
        std::vector<std::thread> ts;
        for (int t = 0; t < T; ++t)
            ts.emplace_back([&, t] {
                const std::size_t a = n * t / T, b = n * (t + 1) / T;
                for (std::size_t i = a; i < b; ++i) out64[i] = m8[i];
            });
        for (auto& th : ts) th.join();
        double t1 = now();
        ts.clear();
        for (int t = 0; t < T; ++t)
            ts.emplace_back([&, t] {
                const std::size_t a = n * t / T, b = n * (t + 1) / T;
                std::uint32_t s = static_cast<std::uint32_t>(a);
                for (std::size_t i = a; i < b; ++i) { s += d8[i]; out32[i] = s; }
            });
        for (auto& th : ts) th.join();
        double t2 = now();
        std::printf("T=%d rep %d: widen u8->u64 %.1f ms (%.1f GB/s written), delta u8->u32 %.1f ms (%.1f GB/s)\n", T, rep,
                    (t1 - t0) * 1e3, n * 8 / (t1 - t0) / 1e9, (t2 - t1) * 1e3, n * 4 / (t2 - t1) / 1e9);
    }
    return 0;
}

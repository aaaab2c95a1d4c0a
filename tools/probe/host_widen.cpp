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
#include <emmintrin.h>
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
        // the same widen with non-temporal 16-byte stores (no read-for-ownership)
        for (int t = 0; t < T; ++t)
            ts.emplace_back([&, t] {
                std::size_t a = n * t / T;
                const std::size_t b = n * (t + 1) / T;
                while (a < b && (reinterpret_cast<std::uintptr_t>(out64 + a) & 15)) { out64[a] = m8[a]; ++a; }
                const __m128i z = _mm_setzero_si128();
                for (; a + 16 <= b; a += 16) {
                    const __m128i v = _mm_loadu_si128(reinterpret_cast<const __m128i*>(&m8[a]));
                    const __m128i w0 = _mm_unpacklo_epi8(v, z), w1 = _mm_unpackhi_epi8(v, z);
                    const __m128i d0 = _mm_unpacklo_epi16(w0, z), d1 = _mm_unpackhi_epi16(w0, z);
                    const __m128i d2 = _mm_unpacklo_epi16(w1, z), d3 = _mm_unpackhi_epi16(w1, z);
                    __m128i* o = reinterpret_cast<__m128i*>(out64 + a);
                    _mm_stream_si128(o + 0, _mm_unpacklo_epi32(d0, z));
                    _mm_stream_si128(o + 1, _mm_unpackhi_epi32(d0, z));
                    _mm_stream_si128(o + 2, _mm_unpacklo_epi32(d1, z));
                    _mm_stream_si128(o + 3, _mm_unpackhi_epi32(d1, z));
                    _mm_stream_si128(o + 4, _mm_unpacklo_epi32(d2, z));
                    _mm_stream_si128(o + 5, _mm_unpackhi_epi32(d2, z));
                    _mm_stream_si128(o + 6, _mm_unpacklo_epi32(d3, z));
                    _mm_stream_si128(o + 7, _mm_unpackhi_epi32(d3, z));
                }
                for (; a < b; ++a) out64[a] = m8[a];
                _mm_sfence();
            });
        for (auto& th : ts) th.join();
        double t1b = now();
        for (std::size_t i = 0; i < n; i += 997)
            if (out64[i] != m8[i]) { std::printf("MISMATCH at %zu\n", i); break; }
        std::printf("   nt-store widen %.1f ms (%.1f GB/s written)\n", (t1b - t1) * 1e3, n * 8 / (t1b - t1) / 1e9);
        t1 = now();
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

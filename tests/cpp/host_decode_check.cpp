// CPU check of the host decoders of the narrow deliveries (csrc/host_decode.hpp)
// against scalar restatements: random steps with escapes, odd lengths, misaligned
// outputs.  Built and run by tests/test_host_decode.py.
#include <cstdio>
#include <random>
#include <vector>

#include "host_decode.hpp"

int main() {
    std::mt19937 rng(7);
    for (int trial = 0; trial < 400; ++trial) {
        const std::size_t n = 1 + rng() % 5000, off = rng() % 4;
        std::vector<std::uint32_t> src(n);
        std::uint32_t v = rng() % 1000;
        for (std::size_t i = 0; i < n; ++i) {
            const int r = static_cast<int>(rng() % 100);
            v += r < 80 ? rng() % 5 : (r < 95 ? rng() % 254 : rng() % 100000);
            src[i] = v;
        }
        // the encoding of k_pack_src for one chunk [0, n): steps, 255 + absolute value
        std::vector<std::uint8_t> d(n, 0);
        std::vector<std::uint32_t> buf(n + 8, 0);
        std::uint32_t* out = buf.data() + off;
        for (std::size_t i = 1; i < n; ++i) {
            const std::uint32_t s = src[i] - src[i - 1];
            if (s > 254) {
                d[i] = 255;
                out[i] = src[i];  // the escape, placed before decoding
            } else {
                d[i] = static_cast<std::uint8_t>(s);
            }
        }
        msc3d_host::decode_steps(d.data(), src[0], out, 0, n);
        _mm_sfence();
        for (std::size_t i = 0; i < n; ++i)
            if (out[i] != src[i]) {
                std::printf("decode_steps: trial %d n %zu off %zu: out[%zu] = %u, want %u\n", trial, n, off, i, out[i],
                            src[i]);
                return 1;
            }
        std::vector<std::uint8_t> m8(n);
        std::vector<std::uint64_t> wide(n + 4, ~0ull);
        std::uint64_t* o64 = wide.data() + (off & 1);
        for (std::size_t i = 0; i < n; ++i) m8[i] = static_cast<std::uint8_t>(rng() % 256);
        const std::size_t a = rng() % n, b = a + rng() % (n - a + 1);
        msc3d_host::widen_u8_u64(m8.data(), o64, a, b);
        for (std::size_t i = 0; i < n; ++i)
            if (o64[i] != (i >= a && i < b ? m8[i] : ~0ull)) {
                std::printf("widen_u8_u64: trial %d: out[%zu] wrong\n", trial, i);
                return 1;
            }
    }
    std::printf("host decoders ok\n");
    return 0;
}

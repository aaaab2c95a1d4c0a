// Canonical synthetic inputs for the BASELINE configs: a seeded
// sum of 32 Gaussians ("gauss"), the same plus 0.01 white noise ("gnoise"), and
// uniform white noise ("noise"), written as f32 x-fastest.  Input generation only;
// nothing here is on the timed path.  The uniform draw is the reference test
// suite's: mt19937_64, (r() >> 11) * 2^-53 (proj/tests/oracles.hpp:45-47).
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <thread>
#include <vector>

namespace {

struct Blob {
    double cx, cy, cz, sigma, amp;
};

inline double unit(std::mt19937_64& r) { return static_cast<double>(r() >> 11) * 0x1.0p-53; }

}  // namespace

extern "C" int msc3d_synth_f32(const char* kind, std::int64_t nx, std::int64_t ny, std::int64_t nz,
                               std::uint64_t seed, float* out, int threads) {
    const bool noise = std::strcmp(kind, "noise") == 0;
    const bool gnoise = std::strcmp(kind, "gnoise") == 0;
    const bool gauss = std::strcmp(kind, "gauss") == 0;
    if (!(noise || gnoise || gauss) || nx < 1 || ny < 1 || nz < 1) return 1;

    std::mt19937_64 rng(seed);
    Blob blob[32];
    for (Blob& b : blob) {
        b.cx = unit(rng) * static_cast<double>(nx);
        b.cy = unit(rng) * static_cast<double>(ny);
        b.cz = unit(rng) * static_cast<double>(nz);
        b.sigma = 0.05 * static_cast<double>(nx) * (0.5 + unit(rng));
        b.amp = 0.5 + unit(rng);
    }
    const std::uint64_t n = static_cast<std::uint64_t>(nx) * ny * nz;
    if (noise) {
        for (std::uint64_t i = 0; i < n; ++i) out[i] = static_cast<float>(unit(rng));
        return 0;
    }
    // The per-vertex noise draws are sequential; precompute them so the Gaussian
    // sums can run on all host threads.
    std::vector<double> jitter;
    if (gnoise) {
        jitter.resize(n);
        for (std::uint64_t i = 0; i < n; ++i) jitter[i] = 0.01 * unit(rng);
    }
    if (threads <= 0) threads = static_cast<int>(std::thread::hardware_concurrency());
    if (threads <= 0) threads = 1;
    auto work = [&](std::int64_t z0, std::int64_t z1) {
        for (std::int64_t z = z0; z < z1; ++z)
            for (std::int64_t y = 0; y < ny; ++y)
                for (std::int64_t x = 0; x < nx; ++x) {
                    double v = 0.0;
                    for (const Blob& b : blob) {
                        const double dx = static_cast<double>(x) - b.cx;
                        const double dy = static_cast<double>(y) - b.cy;
                        const double dz = static_cast<double>(z) - b.cz;
                        v += b.amp * std::exp(-(dx * dx + dy * dy + dz * dz) /
                                              (2.0 * b.sigma * b.sigma));
                    }
                    const std::uint64_t i = static_cast<std::uint64_t>(x) + nx * (y + ny * z);
                    if (gnoise) v += jitter[i];
                    out[i] = static_cast<float>(v);
                }
    };
    std::vector<std::thread> pool;
    const std::int64_t per = (nz + threads - 1) / threads;
    for (int t = 0; t < threads; ++t) {
        const std::int64_t z0 = t * per, z1 = std::min<std::int64_t>(nz, z0 + per);
        if (z0 >= z1) break;
        pool.emplace_back(work, z0, z1);
    }
    for (auto& th : pool) th.join();
    return 0;
}

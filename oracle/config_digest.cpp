// Test infrastructure (oracle/): run the UNMODIFIED reference library once on a raw
// f32 volume and write SHA-256 digests of every output the north star asks to be
// bit-exact: GradientField::code bytes, the four critical-cell lists,
// the critical points (cell, index, value), the sorted arcs with multiplicities, both
// label volumes and input_hash.  Used for the BASELINE configs too large to run live
// inside a GPU test (config 3 = 512^3 gnoise: ~40 min and ~43 GB on 8 cores); the
// digests are committed under tests/golden/ and the -m gpu test hashes the device's
// outputs the same way (tests/test_gpu_configs.py).
//
//   config_digest <raw f32 LE path> nx ny nz threads <out.json>
//
// Reference calls: assign_gradient (gradient.cpp:269-283), extract_critical_cells
// (gradient.cpp:285-297), compute (msc.cpp:57-147), field_hash (msc.cpp:31-42).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <string>
#include <vector>

#include "msc3d/gradient.hpp"
#include "msc3d/grid.hpp"
#include "msc3d/msc.hpp"
#include "sha256.hpp"

using namespace msc3d;
using oracle_sha::digest_of;

namespace {
double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
        .count();
}
}  // namespace

int main(int argc, char** argv) {
    if (argc != 7) {
        std::fprintf(stderr, "usage: %s raw.f32 nx ny nz threads out.json\n", argv[0]);
        return 1;
    }
    const std::int64_t nx = std::atoll(argv[2]), ny = std::atoll(argv[3]), nz = std::atoll(argv[4]);
    const int threads = std::atoi(argv[5]);
    GridDims dims(nx, ny, nz);
    const std::uint64_t V = dims.vertex_count();
    std::vector<float> raw(V);
    {
        std::ifstream in(argv[1], std::ios::binary);
        in.read(reinterpret_cast<char*>(raw.data()), static_cast<std::streamsize>(V * 4));
        if (!in) {
            std::fprintf(stderr, "short read\n");
            return 2;
        }
    }
    ScalarField f(dims, std::vector<double>(raw.begin(), raw.end()));
    raw = std::vector<float>();

    std::string out = "{\n";
    auto kv = [&](const std::string& k, const std::string& v, bool quote) {
        out += "  \"" + k + "\": " + (quote ? "\"" + v + "\"" : v) + ",\n";
    };
    kv("dims", "[" + std::to_string(nx) + ", " + std::to_string(ny) + ", " + std::to_string(nz) + "]",
       false);
    kv("threads", std::to_string(threads), false);

    double t0 = now();
    {
        GradientField g = assign_gradient(f, threads);
        kv("gradient_seconds", std::to_string(now() - t0), false);
        kv("codes", digest_of(g.code.data(), g.code.size()), true);
        const CriticalCells c = extract_critical_cells(g, threads);
        for (int k = 0; k < 4; ++k) {
            kv("crit" + std::to_string(k), digest_of(c.by_dim[k].data(), c.by_dim[k].size()), true);
            kv("n_crit" + std::to_string(k), std::to_string(c.by_dim[k].size()), false);
        }
    }
    std::fprintf(stderr, "gradient + critical digested (%.1f s)\n", now() - t0);

    StageTimings t;
    ComputeOptions opt;
    opt.threads = threads;
    opt.with_segmentation = true;
    opt.source_dtype = "f32";
    opt.timings = &t;
    t0 = now();
    const MSComplex m = compute(f, opt);
    const double wall = now() - t0;
    t0 = now();
    (void)field_hash(f);
    const double hash_s = now() - t0;
    std::fprintf(stderr, "compute done (%.1f s)\n", wall);

    std::vector<std::uint32_t> cell, src, dst;
    std::vector<std::int32_t> index;
    std::vector<double> value;
    cell.reserve(m.critical_points.size());
    index.reserve(m.critical_points.size());
    value.reserve(m.critical_points.size());
    for (const CriticalPoint& cp : m.critical_points) {
        cell.push_back(cp.cell);
        index.push_back(cp.index);
        value.push_back(cp.value);
    }
    kv("cp_cell", digest_of(cell.data(), cell.size()), true);
    kv("cp_index", digest_of(index.data(), index.size()), true);
    kv("cp_value", digest_of(value.data(), value.size()), true);
    kv("n_cp", std::to_string(cell.size()), false);
    std::vector<std::uint64_t> mult;
    src.reserve(m.arcs.size());
    dst.reserve(m.arcs.size());
    mult.reserve(m.arcs.size());
    std::uint64_t max_mult = 0;
    for (const Arc& a : m.arcs) {
        src.push_back(a.src);
        dst.push_back(a.dst);
        mult.push_back(a.multiplicity);
        max_mult = std::max(max_mult, a.multiplicity);
    }
    kv("arc_src", digest_of(src.data(), src.size()), true);
    kv("arc_dst", digest_of(dst.data(), dst.size()), true);
    kv("arc_mult", digest_of(mult.data(), mult.size()), true);
    kv("n_arcs", std::to_string(src.size()), false);
    kv("max_mult", std::to_string(max_mult), false);
    kv("labels_min", digest_of(m.labels->vertex_to_min.data(), m.labels->vertex_to_min.size()), true);
    kv("labels_max", digest_of(m.labels->cube_to_max.data(), m.labels->cube_to_max.size()), true);
    kv("input_hash", std::to_string(m.input_hash), false);
    kv("stage_seconds",
       "[" + std::to_string(t.gradient) + ", " + std::to_string(t.critical) + ", " +
           std::to_string(t.extrema) + ", " + std::to_string(t.reachability) + ", " +
           std::to_string(t.counting) + "]",
       false);
    kv("compute_wall_seconds", std::to_string(wall), false);
    out += "  \"field_hash_seconds\": " + std::to_string(hash_s) + "\n}\n";
    std::ofstream(argv[6]) << out;
    std::fputs(out.c_str(), stdout);
    return 0;
}

// msc3d -- command-line driver of the B200 build, mirroring the reference CLI
// (proj/tools/msc3d_cli.cpp): the same flags, outputs and exit codes
// (0 ok, 1 usage, 2 i/o, 3 invalid input / failed --check, 4 overflow,
// msc3d_cli.cpp:137-166), on top of the drop-in C++ API (include/msc3d/api.hpp).
// The reference parses flags with CLI11 (not in this image); this is a small
// hand-rolled parser for the same flag set.
//
//   msc3d --input v.raw --dims NX NY NZ [--dtype u8|u16|f32|f64] [--big-endian]
//         --out PATH [--format json|csv] [--labels PREFIX] [--check] [--threads N]
//   msc3d generate --kind gauss|gnoise|noise --dims NX NY NZ --out v.raw [--seed S]
//
// `generate` writes the BASELINE synthetic fields (f32 little-endian, SURVEY.md §8(d)
// generator) -- the reference's own generator kinds (ramp, two-bumps, ...) are out of
// scope.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "msc3d/api.hpp"

extern "C" int msc3d_synth_f32(const char* kind, std::int64_t nx, std::int64_t ny, std::int64_t nz,
                               std::uint64_t seed, float* out, int threads) __attribute__((weak));

namespace {

using namespace msc3d;

struct Usage : std::runtime_error {
    using std::runtime_error::runtime_error;
};

void write_text(const std::string& path, const std::string& bytes) {
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) throw IoError("cannot open '" + path + "' for writing");
    out.write(bytes.data(), static_cast<std::streamsize>(bytes.size()));
    out.flush();
    if (!out) throw IoError("write failed on '" + path + "'");
}

void print_timings(const StageTimings& t) {
    std::fprintf(stderr, "stage         seconds\n");
    std::fprintf(stderr, "gradient      %9.3f\n", t.gradient);
    std::fprintf(stderr, "critical      %9.3f\n", t.critical);
    std::fprintf(stderr, "extrema       %9.3f\n", t.extrema);
    std::fprintf(stderr, "reachability  %9.3f\n", t.reachability);
    std::fprintf(stderr, "counting      %9.3f\n", t.counting);
}

int run_compute(const VolumeSpec& spec, const std::string& out, const std::string& format,
                const std::string& labels_prefix, bool check, int threads) {
    const ScalarField f = read_volume(spec);
    StageTimings timings;
    ComputeOptions opt;
    opt.threads = threads;
    opt.with_segmentation = !labels_prefix.empty();
    opt.validate = check;
    opt.source_dtype = sample_type_name(spec.dtype);
    opt.timings = &timings;
    const MSComplex m = compute(f, opt);
    print_timings(timings);
    std::fprintf(stderr,
                 "critical points: %zu (minima %llu, 1-saddles %llu, 2-saddles %llu, maxima %llu); arcs: %zu\n",
                 m.critical_points.size(), static_cast<unsigned long long>(m.count_by_index(0)),
                 static_cast<unsigned long long>(m.count_by_index(1)),
                 static_cast<unsigned long long>(m.count_by_index(2)),
                 static_cast<unsigned long long>(m.count_by_index(3)), m.arcs.size());
    if (check) {
        bool ok = true;
        if (m.euler() != 1) {
            std::fprintf(stderr, "check: Euler characteristic is %lld, want 1\n", static_cast<long long>(m.euler()));
            ok = false;
        }
        const BoundaryReport report = boundary_check(m);
        if (!report.ok()) {
            std::fprintf(stderr, "check: %zu critical point pairs fail mod-2 boundary consistency\n",
                         report.odd_pairs.size());
            ok = false;
        }
        std::fprintf(stderr, "check: gradient ok, euler %s, boundary %s\n", m.euler() == 1 ? "ok" : "BAD",
                     report.ok() ? "ok" : "BAD");
        if (!ok) return 3;
    }
    if (format == "json") {
        write_text(out, serialize_json(m));
    } else {
        write_text(out + "_critical_points.csv", critical_points_csv(m));
        write_text(out + "_arcs.csv", arcs_csv(m));
    }
    if (!labels_prefix.empty()) {
        write_text(labels_prefix + "_min.raw", label_volume_bytes(m.labels->vertex_to_min));
        write_text(labels_prefix + "_max.raw", label_volume_bytes(m.labels->cube_to_max));
    }
    return 0;
}

int run_generate(const std::string& kind, const std::vector<std::int64_t>& dims, const std::string& out,
                 std::uint64_t seed) {
    if (kind != "gauss" && kind != "gnoise" && kind != "noise") throw Usage("--kind must be gauss, gnoise or noise");
    const GridDims gd(dims[0], dims[1], dims[2]);  // the reference's size checks
    if (!msc3d_synth_f32) throw std::runtime_error("synthesizer library not linked");
    std::vector<float> v(static_cast<std::size_t>(gd.nx * gd.ny * gd.nz));
    if (msc3d_synth_f32(kind.c_str(), gd.nx, gd.ny, gd.nz, seed, v.data(), 0) != 0)
        throw std::runtime_error("synthesis failed");
    write_text(out, std::string(reinterpret_cast<const char*>(v.data()), v.size() * sizeof(float)));
    std::fprintf(stderr, "wrote %s: %s %lldx%lldx%lld f32 little-endian\n", out.c_str(), kind.c_str(),
                 static_cast<long long>(gd.nx), static_cast<long long>(gd.ny), static_cast<long long>(gd.nz));
    return 0;
}

std::int64_t to_int(const std::string& s, const char* flag) {
    char* end = nullptr;
    const long long v = std::strtoll(s.c_str(), &end, 10);
    if (s.empty() || *end) throw Usage(std::string(flag) + ": not an integer: " + s);
    return v;
}

}  // namespace

int main(int argc, char** argv) {
    std::string input, out, format = "json", dtype = "f64", labels_prefix, kind;
    std::vector<std::int64_t> dims;
    bool big_endian = false, check = false, generate = false;
    int threads = 0;
    std::uint64_t seed = 1;
    try {
        int i = 1;
        if (i < argc && std::string(argv[i]) == "generate") {
            generate = true;
            ++i;
        }
        auto need = [&](const char* flag) -> std::string {
            if (i + 1 >= argc) throw Usage(std::string(flag) + " needs a value");
            return argv[++i];
        };
        for (; i < argc; ++i) {
            const std::string a = argv[i];
            if (a == "--help" || a == "-h") {
                std::printf("usage: msc3d --input FILE --dims NX NY NZ --out PATH [--dtype u8|u16|f32|f64] "
                            "[--big-endian] [--format json|csv] [--labels PREFIX] [--check] [--threads N]\n"
                            "       msc3d generate --kind gauss|gnoise|noise --dims NX NY NZ --out FILE [--seed S]\n");
                return 0;
            } else if (a == "--input") {
                input = need("--input");
            } else if (a == "--dims") {
                for (int k = 0; k < 3; ++k) dims.push_back(to_int(need("--dims"), "--dims"));
            } else if (a == "--dtype") {
                dtype = need("--dtype");
                if (dtype != "u8" && dtype != "u16" && dtype != "f32" && dtype != "f64")
                    throw Usage("--dtype must be u8, u16, f32 or f64");
            } else if (a == "--big-endian") {
                big_endian = true;
            } else if (a == "--out") {
                out = need("--out");
            } else if (a == "--format") {
                format = need("--format");
                if (format != "json" && format != "csv") throw Usage("--format must be json or csv");
            } else if (a == "--labels") {
                labels_prefix = need("--labels");
            } else if (a == "--check") {
                check = true;
            } else if (a == "--threads") {
                threads = static_cast<int>(to_int(need("--threads"), "--threads"));
                if (threads < 0) throw Usage("--threads must be >= 0");
            } else if (a == "--seed") {
                seed = static_cast<std::uint64_t>(to_int(need("--seed"), "--seed"));
            } else if (a == "--kind") {
                kind = need("--kind");
            } else {
                throw Usage("unknown argument: " + a);
            }
        }
    } catch (const Usage& e) {
        std::fprintf(stderr, "%s\n", e.what());
        return 1;
    }
    try {
        if (generate) {
            if (kind.empty() || dims.size() != 3 || out.empty()) {
                std::fprintf(stderr, "usage: generate needs --kind, --dims and --out\n");
                return 1;
            }
            return run_generate(kind, dims, out, seed);
        }
        if (input.empty() || out.empty() || dims.size() != 3) {
            std::fprintf(stderr, "usage: need --input, --dims and --out (or the generate subcommand); see --help\n");
            return 1;
        }
        VolumeSpec spec;
        spec.path = input;
        spec.dims = GridDims(dims[0], dims[1], dims[2]);
        spec.dtype = parse_sample_type(dtype);
        spec.big_endian = big_endian;
        return run_compute(spec, out, format, labels_prefix, check, threads);
    } catch (const Usage& e) {
        std::fprintf(stderr, "%s\n", e.what());
        return 1;
    } catch (const IoError& e) {
        std::fprintf(stderr, "i/o error: %s\n", e.what());
        return 2;
    } catch (const std::overflow_error& e) {
        std::fprintf(stderr, "overflow: %s\n", e.what());
        return 4;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "invalid input: %s\n", e.what());
        return 3;
    }
}

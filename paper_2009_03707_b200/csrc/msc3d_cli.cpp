// msc3d -- command-line front end of the B200 build.
//
// Flag set and exit-code contract follow the reference CLI (proj/tools/msc3d_cli.cpp:
// 99-166): 0 ok, 1 usage, 2 i/o, 3 invalid input or a failed --check, 4 path-count
// overflow.  Everything below the argument table is the drop-in C++ API
// (include/msc3d/api.hpp), i.e. the device pipeline.
//
//   msc3d --input v.raw --dims NX NY NZ [--dtype u8|u16|f32|f64] [--big-endian]
//         --out PATH [--format json|csv] [--labels PREFIX] [--check] [--threads N]
//   msc3d generate --kind gauss|gnoise|noise --dims NX NY NZ --out v.raw [--seed S]
//
// `generate` writes the BASELINE synthetic fields (f32 little-endian);
// the reference's own f64 generator kinds are out of scope.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "msc3d/api.hpp"

extern "C" int msc3d_synth_f32(const char* kind, std::int64_t nx, std::int64_t ny, std::int64_t nz,
                               std::uint64_t seed, float* out, int threads) __attribute__((weak));

namespace {

enum Exit : int { kOk = 0, kUsage = 1, kIo = 2, kInvalid = 3, kOverflow = 4 };

struct BadUsage : std::runtime_error {
    using std::runtime_error::runtime_error;
};

struct Options {
    bool generate = false;
    std::string input, out, format = "json", dtype = "f64", labels, kind;
    std::vector<std::int64_t> dims;
    bool big_endian = false, check = false, help = false;
    int threads = 0;
    std::uint64_t seed = 1;
};

std::int64_t parse_int(const std::string& text, const std::string& flag) {
    char* end = nullptr;
    const long long v = std::strtoll(text.c_str(), &end, 10);
    if (text.empty() || *end != '\0') throw BadUsage(flag + ": expected an integer, got '" + text + "'");
    return v;
}

std::string one_of(const std::string& v, const std::vector<std::string>& allowed, const std::string& flag) {
    for (const auto& a : allowed)
        if (v == a) return v;
    std::string list;
    for (const auto& a : allowed) list += (list.empty() ? "" : "|") + a;
    throw BadUsage(flag + " must be " + list);
}

// Table of flags: name -> number of values and the action storing them.
Options parse(int argc, char** argv) {
    Options o;
    using Act = std::function<void(const std::vector<std::string>&)>;
    const std::map<std::string, std::pair<int, Act>> table = {
        {"--input", {1, [&](auto& v) { o.input = v[0]; }}},
        {"--out", {1, [&](auto& v) { o.out = v[0]; }}},
        {"--labels", {1, [&](auto& v) { o.labels = v[0]; }}},
        {"--kind", {1, [&](auto& v) { o.kind = v[0]; }}},
        {"--dtype", {1, [&](auto& v) { o.dtype = one_of(v[0], {"u8", "u16", "f32", "f64"}, "--dtype"); }}},
        {"--format", {1, [&](auto& v) { o.format = one_of(v[0], {"json", "csv"}, "--format"); }}},
        {"--dims", {3, [&](auto& v) { for (const auto& s : v) o.dims.push_back(parse_int(s, "--dims")); }}},
        {"--threads", {1, [&](auto& v) {
             o.threads = static_cast<int>(parse_int(v[0], "--threads"));
             if (o.threads < 0) throw BadUsage("--threads must be >= 0");
         }}},
        {"--seed", {1, [&](auto& v) { o.seed = static_cast<std::uint64_t>(parse_int(v[0], "--seed")); }}},
        {"--big-endian", {0, [&](auto&) { o.big_endian = true; }}},
        {"--check", {0, [&](auto&) { o.check = true; }}},
        {"--help", {0, [&](auto&) { o.help = true; }}},
        {"-h", {0, [&](auto&) { o.help = true; }}},
    };
    int i = 1;
    if (i < argc && std::string(argv[i]) == "generate") {
        o.generate = true;
        ++i;
    }
    while (i < argc) {
        const auto it = table.find(argv[i]);
        if (it == table.end()) throw BadUsage(std::string("unknown argument: ") + argv[i]);
        const int want = it->second.first;
        if (i + want > argc - 1)
            throw BadUsage(it->first + " expects " + std::to_string(want) + " value(s)");
        std::vector<std::string> vals(argv + i + 1, argv + i + 1 + want);
        it->second.second(vals);
        i += 1 + want;
    }
    return o;
}

void save(const std::string& path, const std::string& bytes) {
    std::FILE* fh = std::fopen(path.c_str(), "wb");
    if (!fh) throw msc3d::IoError("cannot create " + path);
    const bool ok = std::fwrite(bytes.data(), 1, bytes.size(), fh) == bytes.size();
    if (std::fclose(fh) != 0 || !ok) throw msc3d::IoError("short write to " + path);
}

int cmd_generate(const Options& o) {
    if (o.kind.empty() || o.dims.size() != 3 || o.out.empty())
        throw BadUsage("generate needs --kind, --dims NX NY NZ and --out");
    one_of(o.kind, {"gauss", "gnoise", "noise"}, "--kind");
    const msc3d::GridDims g(o.dims[0], o.dims[1], o.dims[2]);  // the reference's dimension checks
    if (!msc3d_synth_f32) throw std::runtime_error("libmsc3d_synth not linked");
    std::string raw(static_cast<std::size_t>(g.vertex_count()) * sizeof(float), '\0');
    if (msc3d_synth_f32(o.kind.c_str(), g.nx, g.ny, g.nz, o.seed, reinterpret_cast<float*>(&raw[0]), 0) != 0)
        throw std::runtime_error("field synthesis failed");
    save(o.out, raw);
    std::fprintf(stderr, "generate: %s %lld x %lld x %lld (f32 LE) -> %s\n", o.kind.c_str(),
                 static_cast<long long>(g.nx), static_cast<long long>(g.ny), static_cast<long long>(g.nz),
                 o.out.c_str());
    return kOk;
}

int cmd_compute(const Options& o) {
    if (o.input.empty() || o.out.empty() || o.dims.size() != 3)
        throw BadUsage("need --input FILE --dims NX NY NZ --out PATH (or `generate`); see --help");
    msc3d::VolumeSpec spec;
    spec.path = o.input;
    spec.dims = msc3d::GridDims(o.dims[0], o.dims[1], o.dims[2]);
    spec.dtype = msc3d::parse_sample_type(o.dtype);
    spec.big_endian = o.big_endian;

    msc3d::StageTimings t;
    msc3d::ComputeOptions copt;
    copt.threads = o.threads;
    copt.with_segmentation = !o.labels.empty();
    copt.validate = o.check;
    copt.source_dtype = msc3d::sample_type_name(spec.dtype);
    copt.timings = &t;
    // read_volume + compute; f32 LE files go straight into pinned upload memory
    const msc3d::MSComplex cx = msc3d::compute_volume(spec, copt);

    std::fprintf(stderr, "device stage seconds: gradient %.4f | critical %.4f | extrema %.4f | "
                         "reachability %.4f | counting %.4f\n",
                 t.gradient, t.critical, t.extrema, t.reachability, t.counting);
    std::fprintf(stderr, "complex: %zu critical points [%llu %llu %llu %llu], %zu arcs\n",
                 cx.critical_points.size(), static_cast<unsigned long long>(cx.count_by_index(0)),
                 static_cast<unsigned long long>(cx.count_by_index(1)),
                 static_cast<unsigned long long>(cx.count_by_index(2)),
                 static_cast<unsigned long long>(cx.count_by_index(3)), cx.arcs.size());

    if (o.check) {  // the gradient audit already ran inside compute (validate)
        const bool euler_ok = cx.euler() == 1;
        const msc3d::BoundaryReport br = msc3d::boundary_check(cx);
        std::fprintf(stderr, "check: euler=%lld (%s), mod-2 boundary: %zu odd pairs (%s)\n",
                     static_cast<long long>(cx.euler()), euler_ok ? "ok" : "FAIL", br.odd_pairs.size(),
                     br.ok() ? "ok" : "FAIL");
        if (!euler_ok || !br.ok()) return kInvalid;
    }

    if (o.format == "csv") {
        save(o.out + "_critical_points.csv", msc3d::critical_points_csv(cx));
        save(o.out + "_arcs.csv", msc3d::arcs_csv(cx));
    } else {
        save(o.out, msc3d::serialize_json(cx));
    }
    if (cx.labels) {
        save(o.labels + "_min.raw", msc3d::label_volume_bytes(cx.labels->vertex_to_min));
        save(o.labels + "_max.raw", msc3d::label_volume_bytes(cx.labels->cube_to_max));
    }
    return kOk;
}

const char* kHelp =
    "usage: msc3d --input FILE --dims NX NY NZ --out PATH [--dtype u8|u16|f32|f64] [--big-endian]\n"
    "             [--format json|csv] [--labels PREFIX] [--check] [--threads N]\n"
    "       msc3d generate --kind gauss|gnoise|noise --dims NX NY NZ --out FILE [--seed S]\n";

}  // namespace

int main(int argc, char** argv) {
    Options o;
    try {
        o = parse(argc, argv);
    } catch (const std::exception& e) {
        std::fprintf(stderr, "msc3d: %s\n%s", e.what(), kHelp);
        return kUsage;
    }
    if (o.help) {
        std::fputs(kHelp, stdout);
        return kOk;
    }
    try {
        return o.generate ? cmd_generate(o) : cmd_compute(o);
    } catch (const BadUsage& e) {
        std::fprintf(stderr, "msc3d: %s\n", e.what());
        return kUsage;
    } catch (const msc3d::IoError& e) {
        std::fprintf(stderr, "msc3d: i/o: %s\n", e.what());
        return kIo;
    } catch (const std::overflow_error& e) {
        std::fprintf(stderr, "msc3d: overflow: %s\n", e.what());
        return kOverflow;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "msc3d: %s\n", e.what());
        return kInvalid;
    }
}

// Test infrastructure (oracle/): SHA-256 digests of the MS complex of a grid the
// reference rejects (> 2^32 lattice cells, grid.cpp:17-20) -- BASELINE config 4,
// 1024^3 gauss -- computed by our 64-bit restatement oracle64.cpp (pinned against the
// unmodified reference below 2^32 cells by tests/test_oracle.py and the golden
// fixtures).  The per-vertex lower-star pairing and the forest / root passes run on
// several host threads (each cell is written by exactly one vertex, gradient.cpp:79-283;
// pointer doubling is synchronous); the rest is oracle64's serial code, stage by stage,
// freeing what the next stage does not need (peak ~35 GB at 1024^3).
//
//   config4_digest <raw f32 LE path> nx ny nz threads <out.json>
//
// Digests follow oracle/config_digest.cpp, with 64-bit cell ids (crit lists, cp_cell):
// the layout the device uses for such grids (tests/test_gpu_configs.py).
#include <fstream>
#include <thread>

#include "oracle64.cpp"
#include "sha256.hpp"

using oracle_sha::digest_of;

namespace {

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

template <typename F>
void parallel(int T, u64 n, F&& f) {
    std::vector<std::thread> ts;
    for (int t = 0; t < T; ++t)
        ts.emplace_back([&, t] { f(n * t / T, n * (t + 1) / T); });
    for (auto& th : ts) th.join();
}

std::vector<u64> roots_parallel(std::vector<u64> label, int T, int* rounds) {
    *rounds = 0;
    std::vector<u64> next(label.size());
    for (;;) {  // roots() of oracle64.cpp, each round split across threads
        std::vector<char> ch(T, 0);
        std::vector<std::thread> ts;
        for (int t = 0; t < T; ++t)
            ts.emplace_back([&, t] {
                const u64 a = label.size() * t / T, b = label.size() * (t + 1) / T;
                bool c = false;
                for (u64 i = a; i < b; ++i) {
                    next[i] = label[label[i]];
                    c |= next[i] != label[i];
                }
                ch[t] = c;
            });
        for (auto& th : ts) th.join();
        bool changed = false;
        for (char c : ch) changed |= c != 0;
        if (!changed) break;
        ++*rounds;
        label.swap(next);
    }
    return label;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc != 7) {
        std::fprintf(stderr, "usage: %s raw.f32 nx ny nz threads out.json\n", argv[0]);
        return 1;
    }
    const i64 nx = std::atoll(argv[2]), ny = std::atoll(argv[3]), nz = std::atoll(argv[4]);
    const int T = std::max(1, std::atoi(argv[5]));
    const Lattice L(nx, ny, nz);
    std::string out = "{\n";
    auto kv = [&](const std::string& k, const std::string& v, bool quote) {
        out += "  \"" + k + "\": " + (quote ? "\"" + v + "\"" : v) + ",\n";
        std::fprintf(stderr, "%s = %s\n", k.c_str(), v.c_str());
    };
    kv("dims", "[" + std::to_string(nx) + ", " + std::to_string(ny) + ", " + std::to_string(nz) + "]", false);
    kv("threads", std::to_string(T), false);
    const double t_all = now_s();

    std::vector<double> v(L.verts);
    {
        std::FILE* fp = std::fopen(argv[1], "rb");
        if (!fp) return 2;
        std::vector<float> buf(1 << 24);
        for (u64 at = 0; at < L.verts;) {
            const u64 k = std::min<u64>(buf.size(), L.verts - at);
            if (std::fread(buf.data(), 4, k, fp) != k) return 2;
            for (u64 i = 0; i < k; ++i) v[at + i] = buf[i];
            at += k;
        }
        std::fclose(fp);
    }
    // input_hash: FNV-1a over the widened doubles (msc.cpp:31-42)
    u64 h = 0xcbf29ce484222325ull;
    for (u64 i = 0; i < L.verts; ++i) {
        u64 bits;
        std::memcpy(&bits, &v[i], 8);
        for (int s = 0; s < 64; s += 8) {
            h ^= (bits >> s) & 0xffu;
            h *= 0x100000001b3ull;
        }
    }

    // gradient: vertices split by z-planes across threads
    double t0 = now_s();
    std::vector<u8> code(L.cells, 0);
    parallel(T, u64(nz), [&](u64 za, u64 zb) {
        for (i64 z = i64(za); z < i64(zb); ++z)
            for (i64 y = 0; y < ny; ++y)
                for (i64 x = 0; x < nx; ++x) star_pairing(L, v.data(), x, y, z, code.data());
    });
    kv("gradient_seconds", std::to_string(now_s() - t0), false);
    kv("codes", digest_of(code.data(), code.size()), true);
    const auto crit = critical(L, code.data());
    u64 off[4] = {0, 0, 0, 0};
    for (int k = 0; k < 4; ++k) {
        kv("crit" + std::to_string(k), digest_of(crit[k].data(), crit[k].size()), true);
        kv("n_crit" + std::to_string(k), std::to_string(crit[k].size()), false);
        if (k) off[k] = off[k - 1] + crit[k - 1].size();
    }
    {  // critical points (msc.cpp:94-110): cell, index, value at the max vertex
        std::vector<u64> cells;
        std::vector<std::int32_t> index;
        std::vector<double> value;
        for (int k = 0; k < 4; ++k)
            for (u64 c : crit[k]) {
                cells.push_back(c);
                index.push_back(k);
                u64 vs[8];
                const int n = L.vertices(c, vs);
                u64 best = vs[0];  // max_vertex_of (grid.cpp:129-137)
                for (int j = 1; j < n; ++j)
                    if (v[vs[j]] > v[best] || (v[vs[j]] == v[best] && vs[j] > best)) best = vs[j];
                value.push_back(v[best]);
            }
        kv("cp_cell", digest_of(cells.data(), cells.size()), true);
        kv("cp_index", digest_of(index.data(), index.size()), true);
        kv("cp_value", digest_of(value.data(), value.size()), true);
        kv("n_cp", std::to_string(cells.size()), false);
    }
    v = std::vector<double>();
    auto cp = [&](int dim, u64 cell) { return u32(off[dim] + rank_in(crit[dim], cell)); };

    // extremum forests, roots, saddle-extremum arcs, label volumes
    t0 = now_s();
    int r0 = 0, r3 = 0;
    std::vector<u64> l0 = roots_parallel(forest(L, code.data(), 0), T, &r0);
    std::vector<u64> l3 = roots_parallel(forest(L, code.data(), 3), T, &r3);
    const auto sea = se_arcs(L, code.data(), l0.data(), l3.data());
    {
        std::vector<u32> lab(L.verts);
        parallel(T, L.verts, [&](u64 a, u64 b) {
            for (u64 i = a; i < b; ++i) lab[i] = cp(0, L.vcell(l0[i]));
        });
        kv("labels_min", digest_of(lab.data(), lab.size()), true);
    }
    l0 = std::vector<u64>();
    {
        std::vector<u32> lab(L.cubes);
        parallel(T, L.cubes, [&](u64 a, u64 b) {
            for (u64 i = a; i < b; ++i) {
                const u64 r = L.ccell(l3[i]);
                lab[i] = code[r] == CRIT ? cp(3, r) : 0xffffffffu;
            }
        });
        kv("labels_max", digest_of(lab.data(), lab.size()), true);
    }
    l3 = std::vector<u64>();
    kv("rounds0", std::to_string(r0), false);
    kv("rounds3", std::to_string(r3), false);
    kv("extrema_seconds", std::to_string(now_s() - t0), false);

    // saddle-saddle arcs (saddle_graph.cpp, path_matrix.cpp)
    t0 = now_s();
    std::vector<Conn> conns;
    {
        const Marked mk = mark(L, code.data(), crit[1]);
        const Minor mn = build_minor(L, code.data(), mk);
        conns = count_paths(mn);
    }
    kv("saddle_seconds", std::to_string(now_s() - t0), false);
    struct A {
        u32 s, d;
        u64 m;
    };
    std::vector<A> arcs;
    for (const auto& a : sea) {
        if (L.dim(a.saddle) == 1) arcs.push_back({cp(0, a.extremum), cp(1, a.saddle), a.mult});
        else arcs.push_back({cp(2, a.saddle), cp(3, a.extremum), a.mult});
    }
    for (const auto& c : conns) arcs.push_back({cp(1, c.one), cp(2, c.two), c.paths});
    std::sort(arcs.begin(), arcs.end(), [](const A& x, const A& y) { return x.s != y.s ? x.s < y.s : x.d < y.d; });
    std::vector<u32> as, ad;
    std::vector<u64> am;
    u64 max_mult = 0;
    for (const A& a : arcs) {
        as.push_back(a.s);
        ad.push_back(a.d);
        am.push_back(a.m);
        max_mult = std::max(max_mult, a.m);
    }
    kv("arc_src", digest_of(as.data(), as.size()), true);
    kv("arc_dst", digest_of(ad.data(), ad.size()), true);
    kv("arc_mult", digest_of(am.data(), am.size()), true);
    kv("n_arcs", std::to_string(as.size()), false);
    kv("max_mult", std::to_string(max_mult), false);
    kv("input_hash", std::to_string(h), false);
    out += "  \"wall_seconds\": " + std::to_string(now_s() - t_all) + "\n}\n";
    std::ofstream(argv[6]) << out;
    std::fputs(out.c_str(), stdout);
    return 0;
}

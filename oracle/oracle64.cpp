// TEST INFRASTRUCTURE -- serial CPU restatement of the msc3d pipeline with 64-bit
// cell ids ("oracle64").  It is the checker for grids the reference cannot run
// (> 2^32-1 cells: proj/src/grid.cpp:17-20 throws) and is itself pinned against the
// compiled reference (oracle/_ref) and the reference tests' known answers on every
// grid below that limit (tests/test_oracle.py, tests/golden/).  Never linked into,
// or called by, the product library.
//
// Each function cites the reference code it restates.  The algorithms are written
// for obviousness, not speed: plain loops over the lattice, explicit per-star key
// vectors, depth-first path counting with per-node maps.
#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "bundle.hpp"

using oracle_bundle::Bundle;
using u8 = std::uint8_t;
using u32 = std::uint32_t;
using u64 = std::uint64_t;
using i64 = std::int64_t;

ORACLE_BUNDLE_EXPORTS(orc)

namespace {

constexpr u8 CRIT = 1, FAC = 2, COF = 8;  // gradient.hpp:29-41
constexpr u64 NONE = ~0ull;

struct OverflowError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct InvalidArg : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct CycleError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// ---- lattice (grid.hpp:51-114, grid.cpp:11-79) ------------------------------------
struct Lattice {
    i64 n[3];  // vertices per axis
    i64 e[3];  // 2n-1
    u64 cells, verts, cubes;
    Lattice(i64 nx, i64 ny, i64 nz) {
        if (nx < 2 || ny < 2 || nz < 2) throw InvalidArg("dims must be >= 2");
        n[0] = nx; n[1] = ny; n[2] = nz;
        for (int a = 0; a < 3; ++a) e[a] = 2 * n[a] - 1;
        cells = u64(e[0]) * e[1] * e[2];
        verts = u64(nx) * ny * nz;
        cubes = u64(nx - 1) * (ny - 1) * (nz - 1);
    }
    u64 id(const i64 c[3]) const { return u64(c[0] + e[0] * (c[1] + e[1] * c[2])); }
    void coord(u64 id, i64 c[3]) const {
        c[0] = i64(id % u64(e[0]));
        c[1] = i64((id / u64(e[0])) % u64(e[1]));
        c[2] = i64(id / (u64(e[0]) * u64(e[1])));
    }
    int dim(u64 id) const {
        i64 c[3];
        coord(id, c);
        return int((c[0] & 1) + (c[1] & 1) + (c[2] & 1));
    }
    i64 stride(int a) const { return a == 0 ? 1 : (a == 1 ? e[0] : e[0] * e[1]); }
    u64 vcell(u64 v) const {
        const i64 c[3] = {2 * i64(v % u64(n[0])), 2 * i64((v / u64(n[0])) % u64(n[1])),
                          2 * i64(v / (u64(n[0]) * u64(n[1])))};
        return id(c);
    }
    u64 ccell(u64 q) const {
        const u64 mx = u64(n[0] - 1), my = u64(n[1] - 1);
        const i64 c[3] = {2 * i64(q % mx) + 1, 2 * i64((q / mx) % my) + 1, 2 * i64(q / (mx * my)) + 1};
        return id(c);
    }
    u64 vdense(u64 cell) const {
        i64 c[3];
        coord(cell, c);
        return u64(c[0] / 2 + n[0] * (c[1] / 2 + n[1] * (c[2] / 2)));
    }
    u64 cdense(u64 cell) const {
        i64 c[3];
        coord(cell, c);
        return u64(c[0] / 2 + (n[0] - 1) * (c[1] / 2 + (n[1] - 1) * (c[2] / 2)));
    }
    // cofacets: even axes in x,y,z order, minus side first, clipped (grid.cpp:42-59)
    int cofacets(u64 id_, u64 out[6]) const {
        i64 c[3];
        coord(id_, c);
        int k = 0;
        for (int a = 0; a < 3; ++a) {
            if (c[a] & 1) continue;
            if (c[a] > 0) out[k++] = id_ - u64(stride(a));
            if (c[a] < e[a] - 1) out[k++] = id_ + u64(stride(a));
        }
        return k;
    }
    // corner vertices, x fastest (grid.cpp:61-73)
    int vertices(u64 id_, u64 out[8]) const {
        i64 c[3];
        coord(id_, c);
        int k = 0;
        const int sx = (c[0] & 1) ? 2 : 1, sy = (c[1] & 1) ? 2 : 1, sz = (c[2] & 1) ? 2 : 1;
        for (int dz = 0; dz < sz; ++dz)
            for (int dy = 0; dy < sy; ++dy)
                for (int dx = 0; dx < sx; ++dx)
                    out[k++] = u64((c[0] / 2 + dx) + n[0] * ((c[1] / 2 + dy) + n[1] * (c[2] / 2 + dz)));
        return k;
    }
};

u64 partner(const Lattice& L, u64 c, u8 code) {  // gradient.hpp:51-60
    const int dir = code - (code < COF ? FAC : COF);
    const i64 s = L.stride(dir >> 1);
    return (dir & 1) ? c + u64(s) : c - u64(s);
}
bool facet_paired(u8 k) { return k >= FAC && k < COF; }

// ---- gradient (gradient.cpp:79-283) -------------------------------------------------
// The order key of a cell: its vertex values sorted high->low, then its vertex ids
// sorted high->low, the two lists sorted independently (grid.cpp:91-122).
struct Key {
    std::vector<double> val;
    std::vector<u64> vid;
};
bool key_lt(const Key& a, const Key& b) {
    const size_t m = std::min(a.val.size(), b.val.size());
    for (size_t i = 0; i < m; ++i)
        if (a.val[i] != b.val[i]) return a.val[i] < b.val[i];
    if (a.val.size() != b.val.size()) return a.val.size() < b.val.size();
    for (size_t i = 0; i < m; ++i)
        if (a.vid[i] != b.vid[i]) return a.vid[i] < b.vid[i];
    return false;
}

void star_pairing(const Lattice& L, const double* f, i64 vx, i64 vy, i64 vz, u8* code) {
    const u64 vi = u64(vx + L.n[0] * (vy + L.n[1] * vz));
    const double fv = f[vi];
    // The star: cells of the 3x3x3 lattice block around v whose corner vertices
    // other than v all precede v in (value, id) order.
    struct Cell {
        int off[3];
        int dim;
        u64 id;
        Key key;
        bool done = false;
        bool queued1 = false;
    };
    std::vector<Cell> cells;
    int idx_of[27];
    for (int t = 0; t < 27; ++t) idx_of[t] = -1;
    for (int dz = -1; dz <= 1; ++dz)
        for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx) {
                const int off[3] = {dx, dy, dz};
                bool ok = true;
                std::vector<u64> corner;
                // corners of the cell: v plus every combination of its non-zero offsets
                for (int m = 0; m < 8 && ok; ++m) {
                    int o[3];
                    bool valid = true;
                    for (int a = 0; a < 3; ++a) {
                        const bool use = (m >> a) & 1;
                        if (use && off[a] == 0) valid = false;
                        o[a] = use ? off[a] : 0;
                    }
                    if (!valid) continue;
                    const i64 ux = vx + o[0], uy = vy + o[1], uz = vz + o[2];
                    if (ux < 0 || uy < 0 || uz < 0 || ux >= L.n[0] || uy >= L.n[1] || uz >= L.n[2]) {
                        ok = false;
                        break;
                    }
                    const u64 u = u64(ux + L.n[0] * (uy + L.n[1] * uz));
                    if (u != vi && !(f[u] < fv || (f[u] == fv && u < vi))) ok = false;
                    corner.push_back(u);
                }
                if (!ok) continue;
                Cell c;
                for (int a = 0; a < 3; ++a) c.off[a] = off[a];
                c.dim = (dx != 0) + (dy != 0) + (dz != 0);
                const i64 cc[3] = {2 * vx + dx, 2 * vy + dy, 2 * vz + dz};
                c.id = L.id(cc);
                for (u64 u : corner) {
                    c.key.val.push_back(f[u]);
                    c.key.vid.push_back(u);
                }
                std::sort(c.key.val.rbegin(), c.key.val.rend());
                std::sort(c.key.vid.rbegin(), c.key.vid.rend());
                idx_of[(dx + 1) + 3 * (dy + 1) + 9 * (dz + 1)] = int(cells.size());
                cells.push_back(std::move(c));
            }
    const int centre = idx_of[13];
    if (cells.size() == 1) {
        code[cells[centre].id] = CRIT;
        return;
    }
    auto slot_of = [&](const int o[3]) { return (o[0] + 1) + 3 * (o[1] + 1) + 9 * (o[2] + 1); };
    // in-star facets that contain v: zero one non-zero offset
    auto star_facets = [&](int ci, std::vector<int>& out) {
        out.clear();
        for (int a = 0; a < 3; ++a) {
            if (cells[ci].off[a] == 0) continue;
            int o[3] = {cells[ci].off[0], cells[ci].off[1], cells[ci].off[2]};
            o[a] = 0;
            out.push_back(idx_of[slot_of(o)]);
        }
    };
    auto star_cofacets = [&](int ci, std::vector<int>& out) {
        out.clear();
        for (int a = 0; a < 3; ++a) {
            if (cells[ci].off[a] != 0) continue;
            for (int s = -1; s <= 1; s += 2) {
                int o[3] = {cells[ci].off[0], cells[ci].off[1], cells[ci].off[2]};
                o[a] = s;
                const int j = idx_of[slot_of(o)];
                if (j >= 0) out.push_back(j);
            }
        }
    };
    auto pair_up = [&](int lo, int hi) {  // gradient.cpp:162-174
        for (int a = 0; a < 3; ++a) {
            if (cells[lo].off[a] == cells[hi].off[a]) continue;
            const int sgn = cells[hi].off[a] - cells[lo].off[a];
            code[cells[lo].id] = u8(COF + 2 * a + (sgn > 0));
            code[cells[hi].id] = u8(FAC + 2 * a + (sgn < 0));
            return;
        }
    };
    auto free_facets = [&](int ci) {
        std::vector<int> fs;
        star_facets(ci, fs);
        int n = 0;
        for (int j : fs) n += !cells[j].done;
        return n;
    };
    std::vector<int> q1, q0, tmp;
    auto finish = [&](int ci) {  // gradient.cpp:178-193
        cells[ci].done = true;
        star_cofacets(ci, tmp);
        const std::vector<int> cof = tmp;
        for (int j : cof) {
            if (cells[j].done) continue;
            if (free_facets(j) == 1 && !cells[j].queued1) {
                cells[j].queued1 = true;
                q1.push_back(j);
            }
        }
    };
    auto take_lowest = [&](std::vector<int>& q) {
        int best = -1, at = -1;
        for (int i = 0; i < int(q.size()); ++i) {
            if (cells[q[i]].done) continue;
            if (best < 0 || key_lt(cells[q[i]].key, cells[best].key)) {
                best = q[i];
                at = i;
            }
        }
        if (at >= 0) q.erase(q.begin() + at);
        // lazily drop finished entries
        q.erase(std::remove_if(q.begin(), q.end(), [&](int j) { return cells[j].done; }), q.end());
        return best;
    };
    // vertex pairs with its lowest edge; other edges are critical candidates
    int low_edge = -1;
    for (int i = 0; i < int(cells.size()); ++i)
        if (cells[i].dim == 1 && (low_edge < 0 || key_lt(cells[i].key, cells[low_edge].key))) low_edge = i;
    for (int i = 0; i < int(cells.size()); ++i)
        if (cells[i].dim == 1 && i != low_edge) q0.push_back(i);
    pair_up(centre, low_edge);
    finish(centre);
    finish(low_edge);
    int left = int(cells.size()) - 2;
    while (left > 0) {
        for (;;) {
            const int t = take_lowest(q1);
            if (t < 0) break;
            cells[t].queued1 = false;
            if (free_facets(t) != 1) {
                q0.push_back(t);
                continue;
            }
            std::vector<int> fs;
            star_facets(t, fs);
            int fcell = -1;
            for (int j : fs)
                if (!cells[j].done) fcell = j;
            pair_up(fcell, t);
            finish(fcell);
            finish(t);
            left -= 2;
        }
        if (left == 0) break;
        const int t = take_lowest(q0);
        if (t < 0) throw std::logic_error("oracle64: lower-star expansion stalled");
        code[cells[t].id] = CRIT;
        finish(t);
        --left;
    }
}

std::vector<u8> gradient(const Lattice& L, const double* f) {
    std::vector<u8> code(L.cells, 0);
    for (i64 z = 0; z < L.n[2]; ++z)
        for (i64 y = 0; y < L.n[1]; ++y)
            for (i64 x = 0; x < L.n[0]; ++x) star_pairing(L, f, x, y, z, code.data());
    return code;
}

// ---- critical cells (gradient.cpp:285-297) ------------------------------------------
std::array<std::vector<u64>, 4> critical(const Lattice& L, const u8* code) {
    std::array<std::vector<u64>, 4> out;
    for (u64 c = 0; c < L.cells; ++c)
        if (code[c] == CRIT) out[L.dim(c)].push_back(c);
    return out;
}

// ---- forests and roots (extrema.cpp:43-101) -------------------------------------------
std::vector<u64> forest(const Lattice& L, const u8* code, int dim) {
    if (dim != 0 && dim != 3) throw InvalidArg("build_forest: dim must be 0 or 3");
    const u64 n = dim == 0 ? L.verts : L.cubes;
    std::vector<u64> parent(n);
    for (u64 i = 0; i < n; ++i) {
        const u64 c = dim == 0 ? L.vcell(i) : L.ccell(i);
        if (code[c] == CRIT) {
            parent[i] = i;
        } else if (dim == 0) {
            const u64 e = partner(L, c, code[c]);
            parent[i] = L.vdense(2 * e - c);
        } else {
            const u64 q = partner(L, c, code[c]);
            u64 cof[6];
            const int k = L.cofacets(q, cof);
            parent[i] = k == 1 ? i : L.cdense(cof[0] == c ? cof[1] : cof[0]);
        }
    }
    return parent;
}

std::vector<u64> roots(std::vector<u64> label, int* rounds) {
    *rounds = 0;
    std::vector<u64> next(label.size());
    for (;;) {  // synchronous doubling, counting rounds that changed something
        bool changed = false;
        for (size_t i = 0; i < label.size(); ++i) {
            next[i] = label[label[i]];
            changed |= next[i] != label[i];
        }
        if (!changed) break;
        ++*rounds;
        label.swap(next);
    }
    return label;
}

// ---- saddle-extremum arcs (extrema.cpp:103-148) ------------------------------------------
struct SEArc {
    u64 saddle, extremum;
    u32 mult;
};
std::vector<SEArc> se_arcs(const Lattice& L, const u8* code, const u64* l0, const u64* l3) {
    std::vector<SEArc> out;
    for (u64 c = 0; c < L.cells; ++c) {
        if (code[c] != CRIT) continue;
        const int d = L.dim(c);
        if (d != 1 && d != 2) continue;
        u64 end[2] = {NONE, NONE};
        if (d == 1) {
            u64 vs[8];
            L.vertices(c, vs);
            for (int k = 0; k < 2; ++k) end[k] = L.vcell(l0[vs[k]]);
        } else {
            u64 cof[6];
            const int k = L.cofacets(c, cof);
            for (int j = 0; j < k; ++j) {
                const u64 r = L.ccell(l3[L.cdense(cof[j])]);
                if (code[r] == CRIT) end[j] = r;
            }
        }
        if (end[0] != NONE && end[0] == end[1]) {
            out.push_back({c, end[0], 2});
        } else {
            const u64 lo = std::min(end[0], end[1]), hi = std::max(end[0], end[1]);
            if (lo != NONE) out.push_back({c, lo, 1});
            if (hi != NONE) out.push_back({c, hi, 1});
        }
    }
    return out;
}

// ---- DAG successors, reachability (saddle_graph.cpp:10-86) --------------------------------
struct Succ {
    bool terminal;
    u64 cell;
};
int successors(const Lattice& L, const u8* code, u64 e, Succ out[4]) {
    u64 cof[6];
    const int k = L.cofacets(e, cof);
    int n = 0;
    for (int j = 0; j < k; ++j) {
        const u64 q = cof[j];
        if (code[q] == CRIT) out[n++] = {true, q};
        else if (facet_paired(code[q]) && partner(L, q, code[q]) != e) out[n++] = {false, partner(L, q, code[q])};
    }
    return n;
}

struct Marked {
    std::vector<u8> marked;
    std::vector<u64> ones, twos;
};
Marked mark(const Lattice& L, const u8* code, const std::vector<u64>& sources) {
    Marked m;
    m.marked.assign(L.cells, 0);
    std::vector<u64> stack;
    for (u64 e : sources) {
        if (e >= L.cells || code[e] != CRIT || L.dim(e) != 1)
            throw InvalidArg("mark_reachable: sources must be critical 1-cells");
        if (!m.marked[e]) {
            m.marked[e] = 1;
            stack.push_back(e);
        }
    }
    while (!stack.empty()) {  // depth-first; the reached SET is what matters
        const u64 e = stack.back();
        stack.pop_back();
        Succ s[4];
        const int n = successors(L, code, e, s);
        for (int k = 0; k < n; ++k) {
            if (m.marked[s[k].cell]) continue;
            m.marked[s[k].cell] = 1;
            if (!s[k].terminal) {
                m.marked[partner(L, s[k].cell, code[s[k].cell])] = 1;
                stack.push_back(s[k].cell);
            }
        }
    }
    for (u64 c = 0; c < L.cells; ++c) {
        if (!m.marked[c] || code[c] != CRIT) continue;
        const int d = L.dim(c);
        if (d == 1) m.ones.push_back(c);
        if (d == 2) m.twos.push_back(c);
    }
    return m;
}

// ---- minor (saddle_graph.cpp:121-217) ----------------------------------------------------
struct Edge {
    u32 src, dst;
    u64 mult;
};
struct Minor {
    std::vector<u64> ones, juncs, twos;
    std::vector<Edge> e[4];  // s1_to_j, j_to_j, j_to_s2, s1_to_s2
};
u32 rank_in(const std::vector<u64>& v, u64 c) {
    return u32(std::lower_bound(v.begin(), v.end(), c) - v.begin());
}
Minor build_minor(const Lattice& L, const u8* code, const Marked& mk) {
    Minor mn;
    mn.ones = mk.ones;
    mn.twos = mk.twos;
    for (u64 c = 0; c < L.cells; ++c) {
        if (!mk.marked[c] || code[c] == CRIT || L.dim(c) != 1) continue;
        Succ s[4];
        if (successors(L, code, c, s) > 1) mn.juncs.push_back(c);
    }
    auto is_j = [&](u64 c) { return std::binary_search(mn.juncs.begin(), mn.juncs.end(), c); };
    std::map<std::pair<u32, u32>, u64> acc[4];
    auto trace = [&](bool from_j, u32 origin, Succ s) {
        // walk junction-free cells until a 2-saddle or junction; dead ends vanish
        u64 steps = 0;
        for (;;) {
            if (s.terminal) {
                ++acc[from_j ? 2 : 3][{origin, rank_in(mn.twos, s.cell)}];
                return;
            }
            if (is_j(s.cell)) {
                ++acc[from_j ? 1 : 0][{origin, rank_in(mn.juncs, s.cell)}];
                return;
            }
            Succ nx[4];
            const int n = successors(L, code, s.cell, nx);
            if (n == 0) return;
            s = nx[0];
            if (++steps > L.cells) throw CycleError("build_minor: trace outlived the grid (cycle)");
        }
    };
    for (u32 i = 0; i < mn.ones.size(); ++i) {
        Succ s[4];
        const int n = successors(L, code, mn.ones[i], s);
        for (int k = 0; k < n; ++k) trace(false, i, s[k]);
    }
    for (u32 i = 0; i < mn.juncs.size(); ++i) {
        Succ s[4];
        const int n = successors(L, code, mn.juncs[i], s);
        for (int k = 0; k < n; ++k) trace(true, i, s[k]);
    }
    for (int k = 0; k < 4; ++k)
        for (const auto& kv : acc[k]) mn.e[k].push_back({kv.first.first, kv.first.second, kv.second});
    return mn;
}

// ---- path counting (path_matrix.cpp:188-219) ----------------------------------------------
// The reference raises overflow_error iff some 1-saddle->junction path count
// (an entry of A* = A(I+B+B^2+...)) or some final 1-saddle->2-saddle count leaves
// 64 bits, and runtime_error iff its frontier A*B^k never empties, i.e. a junction
// cycle is reachable from a 1-saddle.  Restated with per-junction count maps
// computed depth-first (P(j)[t] = paths j -> t), plus a forward pass for A*.
struct Conn {
    u64 one, two, paths;
};
bool add_ok(u64 a, u64 b, u64* r) { return !__builtin_add_overflow(a, b, r); }
bool mul_ok(u64 a, u64 b, u64* r) { return !__builtin_mul_overflow(a, b, r); }

std::vector<Conn> count_paths(const Minor& mn) {
    const size_t n1 = mn.ones.size(), nj = mn.juncs.size(), n2 = mn.twos.size();
    for (int k = 0; k < 4; ++k)
        for (const Edge& e : mn.e[k]) {
            const size_t rs = (k == 0 || k == 3) ? n1 : nj, cs = (k == 0 || k == 1) ? nj : n2;
            if (e.src >= rs || e.dst >= cs) throw InvalidArg("from_edges: edge endpoint out of range");
        }
    std::vector<std::vector<std::pair<u32, u64>>> jj(nj), j2(nj), sj(n1), s2(n1);
    // from_edges drops zero sums and sums duplicates (path_matrix.cpp:84-113)
    auto load = [&](const std::vector<Edge>& es, std::vector<std::vector<std::pair<u32, u64>>>& adj) {
        std::map<std::pair<u32, u32>, u64> sum;
        for (const Edge& e : es) {
            u64& s = sum[{e.src, e.dst}];
            if (!add_ok(s, e.mult, &s)) throw OverflowError("from_edges: multiplicity sum exceeds 64 bits");
        }
        for (const auto& kv : sum)
            if (kv.second) adj[kv.first.first].push_back({kv.first.second, kv.second});
    };
    load(mn.e[0], sj);
    load(mn.e[1], jj);
    load(mn.e[2], j2);
    load(mn.e[3], s2);

    // junctions reachable from 1-saddles; a reachable cycle is the runtime_error
    std::vector<u8> reach(nj, 0), color(nj, 0);
    std::vector<u32> stack;
    for (size_t i = 0; i < n1; ++i)
        for (auto& x : sj[i])
            if (!reach[x.first]) {
                reach[x.first] = 1;
                stack.push_back(x.first);
            }
    while (!stack.empty()) {
        const u32 j = stack.back();
        stack.pop_back();
        for (auto& x : jj[j])
            if (!reach[x.first]) {
                reach[x.first] = 1;
                stack.push_back(x.first);
            }
    }
    // topological order of reachable junctions (DFS post-order), cycle check
    std::vector<u32> post;
    for (u32 r = 0; r < nj; ++r) {
        if (!reach[r] || color[r]) continue;
        std::vector<std::pair<u32, size_t>> st{{r, 0}};
        color[r] = 1;
        while (!st.empty()) {
            auto& [j, it] = st.back();
            if (it < jj[j].size()) {
                const u32 nx = jj[j][it++].first;
                if (color[nx] == 1) throw CycleError("count_paths: junction graph has a cycle");
                if (color[nx] == 0) {
                    color[nx] = 1;
                    st.push_back({nx, 0});
                }
            } else {
                color[j] = 2;
                post.push_back(j);
                st.pop_back();
            }
        }
    }
    // forward A*: total paths from all 1-saddles into each junction (saturating);
    // only if a total saturates is the exact per-source count needed.
    std::vector<unsigned __int128> fwd(nj, 0);
    const unsigned __int128 cap = (unsigned __int128)1 << 100;
    auto sat_add = [&](unsigned __int128 a, unsigned __int128 b) { return a + b > cap ? cap : a + b; };
    for (size_t i = 0; i < n1; ++i)
        for (auto& x : sj[i]) fwd[x.first] = sat_add(fwd[x.first], x.second);
    for (size_t p = post.size(); p-- > 0;) {
        const u32 j = post[p];
        for (auto& x : jj[j]) {
            unsigned __int128 t = fwd[j] * x.second;
            if (fwd[j] != 0 && t / fwd[j] != x.second) t = cap;
            fwd[x.first] = sat_add(fwd[x.first], t > cap ? cap : t);
        }
    }
    bool need_exact = false;
    for (u32 j = 0; j < nj; ++j) need_exact |= fwd[j] > ~0ull;
    if (need_exact) {
        for (size_t i = 0; i < n1; ++i) {  // exact per source, topological order
            std::vector<unsigned __int128> a(nj, 0);
            for (auto& x : sj[i]) a[x.first] += x.second;
            for (size_t p = post.size(); p-- > 0;) {
                const u32 j = post[p];
                if (a[j] > ~0ull) throw OverflowError("count_paths: path count exceeds 64 bits");
                for (auto& x : jj[j]) {
                    unsigned __int128 t = a[j] * x.second;
                    if (a[j] != 0 && t / a[j] != x.second) t = cap;
                    a[x.first] = sat_add(a[x.first], t > cap ? cap : t);
                }
            }
        }
    }
    // backward: P(j) in post-order (successors first)
    std::vector<std::map<u32, u64>> P(nj);
    for (u32 j : post) {
        std::map<u32, u64> s;
        for (auto& x : j2[j]) {
            u64& v = s[x.first];
            if (!add_ok(v, x.second, &v)) throw OverflowError("count_paths: path count exceeds 64 bits");
        }
        for (auto& x : jj[j])
            for (auto& y : P[x.first]) {
                u64 t;
                if (!mul_ok(y.second, x.second, &t)) throw OverflowError("count_paths: path count exceeds 64 bits");
                u64& v = s[y.first];
                if (!add_ok(v, t, &v)) throw OverflowError("count_paths: path count exceeds 64 bits");
            }
        P[j] = std::move(s);
    }
    std::vector<Conn> out;
    for (size_t i = 0; i < n1; ++i) {
        std::map<u32, u64> s;
        for (auto& x : s2[i]) {
            u64& v = s[x.first];
            if (!add_ok(v, x.second, &v)) throw OverflowError("count_paths: path count exceeds 64 bits");
        }
        for (auto& x : sj[i])
            for (auto& y : P[x.first]) {
                u64 t;
                if (!mul_ok(y.second, x.second, &t)) throw OverflowError("count_paths: path count exceeds 64 bits");
                u64& v = s[y.first];
                if (!add_ok(v, t, &v)) throw OverflowError("count_paths: path count exceeds 64 bits");
            }
        for (auto& kv : s)
            if (kv.second) out.push_back({mn.ones[i], mn.twos[kv.first], kv.second});
    }
    return out;
}

template <typename Fn>
void* guarded(Fn&& fn) {
    auto* b = new Bundle();
    try {
        fn(*b);
    } catch (const InvalidArg& e) {
        b->status = 1;
        b->error = e.what();
    } catch (const OverflowError& e) {
        b->status = 2;
        b->error = e.what();
    } catch (const CycleError& e) {
        b->status = 3;
        b->error = e.what();
    } catch (const std::exception& e) {
        b->status = 4;
        b->error = e.what();
    }
    return b;
}

void put_minor(Bundle& b, const Minor& mn) {
    b.put("one_saddles", mn.ones);
    b.put("junctions", mn.juncs);
    b.put("two_saddles", mn.twos);
    const char* names[4] = {"s1_to_j", "j_to_j", "j_to_s2", "s1_to_s2"};
    for (int k = 0; k < 4; ++k) {
        std::vector<u32> s, t;
        std::vector<u64> m;
        for (const Edge& e : mn.e[k]) {
            s.push_back(e.src);
            t.push_back(e.dst);
            m.push_back(e.mult);
        }
        b.put(std::string(names[k]) + ".src", s);
        b.put(std::string(names[k]) + ".dst", t);
        b.put(std::string(names[k]) + ".mult", m);
    }
}

}  // namespace

extern "C" {

void* orc_gradient(const double* v, i64 nx, i64 ny, i64 nz, int) {
    return guarded([&](Bundle& b) {
        const Lattice L(nx, ny, nz);
        for (u64 i = 0; i < L.verts; ++i)
            if (!std::isfinite(v[i])) throw InvalidArg("scalar field contains a non-finite value");
        b.put("codes", gradient(L, v));
    });
}

void* orc_critical(const u8* code, i64 nx, i64 ny, i64 nz, int) {
    return guarded([&](Bundle& b) {
        const Lattice L(nx, ny, nz);
        auto c = critical(L, code);
        for (int k = 0; k < 4; ++k) b.put("c" + std::to_string(k), c[k]);
    });
}

void* orc_forest(const u8* code, i64 nx, i64 ny, i64 nz, int dim, int) {
    return guarded([&](Bundle& b) { b.put("parent", forest(Lattice(nx, ny, nz), code, dim)); });
}

void* orc_roots(const u64* parent, u64 n, int) {
    return guarded([&](Bundle& b) {
        int rounds = 0;
        b.put("label", roots(std::vector<u64>(parent, parent + n), &rounds));
        b.put_scalar<std::int32_t>("rounds", rounds);
    });
}

void* orc_se_arcs(const u8* code, i64 nx, i64 ny, i64 nz, const u64* l0, const u64* l3, int) {
    return guarded([&](Bundle& b) {
        const auto arcs = se_arcs(Lattice(nx, ny, nz), code, l0, l3);
        std::vector<u64> s, e;
        std::vector<u32> m;
        for (const auto& a : arcs) {
            s.push_back(a.saddle);
            e.push_back(a.extremum);
            m.push_back(a.mult);
        }
        b.put("saddle", s);
        b.put("extremum", e);
        b.put("mult", m);
    });
}

void* orc_mark(const u8* code, i64 nx, i64 ny, i64 nz, const u64* src, u64 n, int) {
    return guarded([&](Bundle& b) {
        const Marked m = mark(Lattice(nx, ny, nz), code, std::vector<u64>(src, src + n));
        b.put("marked", m.marked);
        b.put("one_saddles", m.ones);
        b.put("two_saddles", m.twos);
    });
}

void* orc_minor(const u8* code, i64 nx, i64 ny, i64 nz, const u8* marked, const u64* ones, u64 n1,
                const u64* twos, u64 n2, int) {
    return guarded([&](Bundle& b) {
        const Lattice L(nx, ny, nz);
        Marked m;
        m.marked.assign(marked, marked + L.cells);
        m.ones.assign(ones, ones + n1);
        m.twos.assign(twos, twos + n2);
        put_minor(b, build_minor(L, code, m));
    });
}

void* orc_count_paths(const u64* ones, u64 n1, const u64* juncs, u64 nj, const u64* twos, u64 n2,
                      const u32* const* src, const u32* const* dst, const u64* const* mult,
                      const u64* count, int) {
    return guarded([&](Bundle& b) {
        Minor mn;
        mn.ones.assign(ones, ones + n1);
        mn.juncs.assign(juncs, juncs + nj);
        mn.twos.assign(twos, twos + n2);
        for (int k = 0; k < 4; ++k)
            for (u64 i = 0; i < count[k]; ++i) mn.e[k].push_back({src[k][i], dst[k][i], mult[k][i]});
        const auto out = count_paths(mn);
        std::vector<u64> a, c, p;
        for (const Conn& x : out) {
            a.push_back(x.one);
            c.push_back(x.two);
            p.push_back(x.paths);
        }
        b.put("one_saddle", a);
        b.put("two_saddle", c);
        b.put("paths", p);
    });
}

// compute() (msc.cpp:57-147) with segmentation; ids are 64-bit here, arcs u32 cp ids.
void* orc_compute(const double* v, i64 nx, i64 ny, i64 nz, int, int with_seg, int, const char*, int) {
    return guarded([&](Bundle& b) {
        const Lattice L(nx, ny, nz);
        for (u64 i = 0; i < L.verts; ++i)
            if (!std::isfinite(v[i])) throw InvalidArg("scalar field contains a non-finite value");
        const auto t0 = std::chrono::steady_clock::now();
        const std::vector<u8> code = gradient(L, v);
        const auto crit = critical(L, code.data());
        int r0 = 0, r3 = 0;
        const auto l0 = roots(forest(L, code.data(), 0), &r0);
        const auto l3 = roots(forest(L, code.data(), 3), &r3);
        const auto sea = se_arcs(L, code.data(), l0.data(), l3.data());
        const Marked mk = mark(L, code.data(), crit[1]);
        const Minor mn = build_minor(L, code.data(), mk);
        const auto conns = count_paths(mn);
        const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();

        u64 off[4] = {0, 0, 0, 0};
        for (int k = 1; k < 4; ++k) off[k] = off[k - 1] + crit[k - 1].size();
        auto cp = [&](int dim, u64 cell) { return u32(off[dim] + rank_in(crit[dim], cell)); };
        std::vector<u64> cells;
        std::vector<std::int32_t> index;
        std::vector<double> value;
        for (int k = 0; k < 4; ++k)
            for (u64 c : crit[k]) {
                cells.push_back(c);
                index.push_back(k);
                u64 vs[8];
                const int nv = L.vertices(c, vs);
                u64 best = vs[0];  // max_vertex_of (grid.cpp:129-137)
                for (int j = 1; j < nv; ++j)
                    if (v[vs[j]] > v[best] || (v[vs[j]] == v[best] && vs[j] > best)) best = vs[j];
                value.push_back(v[best]);
            }
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
        std::sort(arcs.begin(), arcs.end(), [](const A& x, const A& y) {
            return x.s != y.s ? x.s < y.s : x.d < y.d;
        });
        std::vector<u32> as, ad;
        std::vector<u64> am;
        for (const A& a : arcs) {
            as.push_back(a.s);
            ad.push_back(a.d);
            am.push_back(a.m);
        }
        b.put("cp_cell", cells);
        b.put("cp_index", index);
        b.put("cp_value", value);
        b.put("arc_src", as);
        b.put("arc_dst", ad);
        b.put("arc_mult", am);
        // FNV-1a over the widened doubles (msc.cpp:31-42)
        u64 h = 0xcbf29ce484222325ull;
        for (u64 i = 0; i < L.verts; ++i) {
            u64 bits;
            std::memcpy(&bits, &v[i], 8);
            for (int s = 0; s < 64; s += 8) {
                h ^= (bits >> s) & 0xffu;
                h *= 0x100000001b3ull;
            }
        }
        b.put_scalar<u64>("input_hash", h);
        b.put("timings", std::vector<double>{0, 0, 0, 0, 0});
        b.put_scalar("wall", wall);
        b.put_scalar("hash_seconds", 0.0);
        if (with_seg) {
            std::vector<u32> lmin(L.verts), lmax(L.cubes);
            for (u64 i = 0; i < L.verts; ++i) lmin[i] = cp(0, L.vcell(l0[i]));
            for (u64 i = 0; i < L.cubes; ++i) {
                const u64 r = L.ccell(l3[i]);
                lmax[i] = code[r] == CRIT ? cp(3, r) : 0xffffffffu;
            }
            b.put("labels_min", lmin);
            b.put("labels_max", lmax);
        }
    });
}

}  // extern "C"

// Test infrastructure (oracle/): flat extern "C" harness over the UNMODIFIED
// reference library (/root/reference/proj/src, compiled by oracle/Makefile into
// oracle/_ref/).  Every entry point forwards to one reference function and returns
// its outputs as a Bundle of named arrays; exceptions become Bundle::status codes
// (1 invalid_argument, 2 overflow_error, 3 runtime_error, 4 other, 5 IoError).
//
// This is the checker the GPU parity tests and bench.py's reference/cpu_baseline
// arm call.  It is never linked into the product (paper_2009_03707_b200/).
#include <chrono>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "bundle.hpp"
#include "msc3d/extrema.hpp"
#include "msc3d/gradient.hpp"
#include "msc3d/grid.hpp"
#include "msc3d/msc.hpp"
#include "msc3d/path_matrix.hpp"
#include "msc3d/saddle_graph.hpp"
#include "msc3d/serialize.hpp"
#include "msc3d/volume.hpp"

using oracle_bundle::Bundle;
using namespace msc3d;

ORACLE_BUNDLE_EXPORTS(ref)

namespace {

template <typename Fn>
void* guarded(Fn&& fn) {
    auto* b = new Bundle();
    try {
        fn(*b);
    } catch (const IoError& e) {
        b->status = 5;
        b->error = e.what();
    } catch (const std::invalid_argument& e) {
        b->status = 1;
        b->error = e.what();
    } catch (const std::overflow_error& e) {
        b->status = 2;
        b->error = e.what();
    } catch (const std::runtime_error& e) {
        b->status = 3;
        b->error = e.what();
    } catch (const std::exception& e) {
        b->status = 4;
        b->error = e.what();
    }
    return b;
}

GradientField make_gradient(const std::uint8_t* codes, std::int64_t nx, std::int64_t ny,
                            std::int64_t nz) {
    GridDims d(nx, ny, nz);
    return GradientField{d, std::vector<std::uint8_t>(codes, codes + d.total_cells())};
}

void put_edges(Bundle& b, const std::string& name, const std::vector<MinorEdge>& es) {
    std::vector<std::uint32_t> s, t;
    std::vector<std::uint64_t> m;
    for (const MinorEdge& e : es) {
        s.push_back(e.src);
        t.push_back(e.dst);
        m.push_back(e.multiplicity);
    }
    b.put(name + ".src", s);
    b.put(name + ".dst", t);
    b.put(name + ".mult", m);
}

std::vector<MinorEdge> get_edges(const std::uint32_t* s, const std::uint32_t* t,
                                 const std::uint64_t* m, std::uint64_t n) {
    std::vector<MinorEdge> out(n);
    for (std::uint64_t i = 0; i < n; ++i) out[i] = MinorEdge{s[i], t[i], m[i]};
    return out;
}

}  // namespace

extern "C" {

int ref_dims_ok(std::int64_t nx, std::int64_t ny, std::int64_t nz) {
    try {
        GridDims d(nx, ny, nz);
        return 0;
    } catch (const std::invalid_argument&) {
        return 1;
    }
}

void* ref_gradient(const double* values, std::int64_t nx, std::int64_t ny, std::int64_t nz,
                   int threads) {
    return guarded([&](Bundle& b) {
        GridDims d(nx, ny, nz);
        ScalarField f(d, std::vector<double>(values, values + d.vertex_count()));
        const auto t0 = std::chrono::steady_clock::now();
        GradientField g = assign_gradient(f, threads);
        const double secs =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        b.put("codes", g.code);
        b.put_scalar("seconds", secs);
    });
}

void* ref_validate_gradient(const std::uint8_t* codes, std::int64_t nx, std::int64_t ny,
                            std::int64_t nz, std::uint64_t max_cells_for_cycles) {
    return guarded([&](Bundle& b) {
        const GradientReport r = validate_gradient(make_gradient(codes, nx, ny, nz), max_cells_for_cycles);
        b.put_scalar<std::uint64_t>("matching_violations", r.matching_violations);
        b.put_scalar<std::uint64_t>("cells_in_closed_vpath", r.cells_in_closed_vpath);
        b.put_scalar<std::uint8_t>("acyclicity_checked", r.acyclicity_checked);
        b.put_scalar<std::uint8_t>("degenerate", r.degenerate);
    });
}

void* ref_critical(const std::uint8_t* codes, std::int64_t nx, std::int64_t ny, std::int64_t nz,
                   int threads) {
    return guarded([&](Bundle& b) {
        const CriticalCells c = extract_critical_cells(make_gradient(codes, nx, ny, nz), threads);
        for (int k = 0; k < 4; ++k) b.put("c" + std::to_string(k), c.by_dim[k]);
    });
}

void* ref_forest(const std::uint8_t* codes, std::int64_t nx, std::int64_t ny, std::int64_t nz,
                 int dim, int threads) {
    return guarded([&](Bundle& b) {
        const ParentForest f = build_forest(make_gradient(codes, nx, ny, nz), dim, threads);
        b.put("parent", f.parent);
    });
}

void* ref_roots(const std::uint32_t* parent, std::uint64_t n, int threads) {
    return guarded([&](Bundle& b) {
        ParentForest f;
        f.parent.assign(parent, parent + n);
        const RootLabels r = find_roots(f, threads);
        b.put("label", r.label);
        b.put_scalar<std::int32_t>("rounds", r.rounds);
    });
}

void* ref_se_arcs(const std::uint8_t* codes, std::int64_t nx, std::int64_t ny, std::int64_t nz,
                  const std::uint32_t* l0, const std::uint32_t* l3, int threads) {
    return guarded([&](Bundle& b) {
        const GradientField g = make_gradient(codes, nx, ny, nz);
        RootLabels r0, r3;
        r0.label.assign(l0, l0 + g.dims.vertex_count());
        r3.label.assign(l3, l3 + g.dims.cube_count());
        const auto arcs = saddle_extremum_arcs(g, r0, r3, threads);
        std::vector<std::uint32_t> s, e, m;
        for (const auto& a : arcs) {
            s.push_back(a.saddle);
            e.push_back(a.extremum);
            m.push_back(a.multiplicity);
        }
        b.put("saddle", s);
        b.put("extremum", e);
        b.put("mult", m);
    });
}

void* ref_successors(const std::uint8_t* codes, std::int64_t nx, std::int64_t ny,
                     std::int64_t nz, std::uint32_t edge) {
    return guarded([&](Bundle& b) {
        const SuccessorList ss = successors(make_gradient(codes, nx, ny, nz), edge);
        std::vector<std::uint8_t> kind;
        std::vector<std::uint32_t> cell;
        for (int k = 0; k < ss.count; ++k) {
            kind.push_back(static_cast<std::uint8_t>(ss[k].kind));
            cell.push_back(ss[k].cell);
        }
        b.put("kind", kind);
        b.put("cell", cell);
    });
}

void* ref_mark(const std::uint8_t* codes, std::int64_t nx, std::int64_t ny, std::int64_t nz,
               const std::uint32_t* sources, std::uint64_t nsrc, int threads) {
    return guarded([&](Bundle& b) {
        const MarkedSubgraph m = mark_reachable(make_gradient(codes, nx, ny, nz),
                                                std::vector<CellIndex>(sources, sources + nsrc),
                                                threads);
        b.put("marked", m.marked);
        b.put("one_saddles", m.one_saddles);
        b.put("two_saddles", m.two_saddles);
    });
}

void* ref_minor(const std::uint8_t* codes, std::int64_t nx, std::int64_t ny, std::int64_t nz,
                const std::uint8_t* marked, const std::uint32_t* ones, std::uint64_t n1,
                const std::uint32_t* twos, std::uint64_t n2, int threads) {
    return guarded([&](Bundle& b) {
        const GradientField g = make_gradient(codes, nx, ny, nz);
        MarkedSubgraph m;
        m.dims = g.dims;
        m.marked.assign(marked, marked + g.dims.total_cells());
        m.one_saddles.assign(ones, ones + n1);
        m.two_saddles.assign(twos, twos + n2);
        const DagMinor mn = build_minor(m, g, threads);
        b.put("one_saddles", mn.one_saddles);
        b.put("junctions", mn.junctions);
        b.put("two_saddles", mn.two_saddles);
        put_edges(b, "s1_to_j", mn.s1_to_j);
        put_edges(b, "j_to_j", mn.j_to_j);
        put_edges(b, "j_to_s2", mn.j_to_s2);
        put_edges(b, "s1_to_s2", mn.s1_to_s2);
    });
}

// Edge lists are passed as 4 x (src*, dst*, mult*, n) in the order
// s1_to_j, j_to_j, j_to_s2, s1_to_s2.
void* ref_count_paths(const std::uint32_t* ones, std::uint64_t n1, const std::uint32_t* juncs,
                      std::uint64_t nj, const std::uint32_t* twos, std::uint64_t n2,
                      const std::uint32_t* const* src, const std::uint32_t* const* dst,
                      const std::uint64_t* const* mult, const std::uint64_t* count, int threads) {
    return guarded([&](Bundle& b) {
        DagMinor m;
        m.one_saddles.assign(ones, ones + n1);
        m.junctions.assign(juncs, juncs + nj);
        m.two_saddles.assign(twos, twos + n2);
        m.s1_to_j = get_edges(src[0], dst[0], mult[0], count[0]);
        m.j_to_j = get_edges(src[1], dst[1], mult[1], count[1]);
        m.j_to_s2 = get_edges(src[2], dst[2], mult[2], count[2]);
        m.s1_to_s2 = get_edges(src[3], dst[3], mult[3], count[3]);
        const auto out = count_paths(m, threads);
        std::vector<std::uint32_t> a, c;
        std::vector<std::uint64_t> p;
        for (const auto& s : out) {
            a.push_back(s.one_saddle);
            c.push_back(s.two_saddle);
            p.push_back(s.paths);
        }
        b.put("one_saddle", a);
        b.put("two_saddle", c);
        b.put("paths", p);
    });
}

std::uint64_t ref_field_hash(const double* values, std::uint64_t n) {
    ScalarField f;
    f.values.assign(values, values + n);
    return field_hash(f);
}

void* ref_read_volume(const char* path, std::int64_t nx, std::int64_t ny, std::int64_t nz,
                      const char* dtype, int big_endian) {
    return guarded([&](Bundle& b) {
        VolumeSpec spec;
        spec.path = path;
        spec.dims = GridDims(nx, ny, nz);
        spec.dtype = parse_sample_type(dtype);
        spec.big_endian = big_endian != 0;
        const ScalarField f = read_volume(spec);
        b.put("values", f.values);
    });
}

void* ref_generate(const char* kind, std::int64_t nx, std::int64_t ny, std::int64_t nz,
                   std::uint64_t seed) {
    return guarded([&](Bundle& b) {
        const ScalarField f = generate_field(parse_field_kind(kind), GridDims(nx, ny, nz), seed);
        b.put("values", f.values);
    });
}

std::uint32_t ref_max_vertex_of(const double* values, std::int64_t nx, std::int64_t ny,
                                std::int64_t nz, std::uint32_t cell) {
    GridDims d(nx, ny, nz);
    ScalarField f(d, std::vector<double>(values, values + d.vertex_count()));
    return max_vertex_of(f, cell);
}

int ref_compare_cells(const double* values, std::int64_t nx, std::int64_t ny, std::int64_t nz,
                      std::uint32_t a, std::uint32_t c) {
    GridDims d(nx, ny, nz);
    ScalarField f(d, std::vector<double>(values, values + d.vertex_count()));
    const auto o = compare_cells(f, a, c);
    return o == std::strong_ordering::less ? -1 : (o == std::strong_ordering::equal ? 0 : 1);
}

// compute(): the whole pipeline plus the writers.  "timings" = the five
// StageTimings fields; "wall" = wall clock around compute(); "hash_seconds" =
// a separate timing of field_hash (the serial FNV-1a compute() runs untimed).
void* ref_compute(const double* values, std::int64_t nx, std::int64_t ny, std::int64_t nz,
                  int threads, int with_segmentation, int validate, const char* dtype,
                  int want_text) {
    return guarded([&](Bundle& b) {
        GridDims d(nx, ny, nz);
        ScalarField f(d, std::vector<double>(values, values + d.vertex_count()));
        StageTimings t;
        ComputeOptions opt;
        opt.threads = threads;
        opt.with_segmentation = with_segmentation != 0;
        opt.validate = validate != 0;
        opt.source_dtype = dtype;
        opt.timings = &t;
        const auto t0 = std::chrono::steady_clock::now();
        const MSComplex m = compute(f, opt);
        const double wall =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        const auto h0 = std::chrono::steady_clock::now();
        (void)field_hash(f);
        const double hash_secs =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - h0).count();

        std::vector<std::uint32_t> cell, aid, src, dst;
        std::vector<std::int32_t> index, doubled;
        std::vector<double> value, midpoint;
        for (const CriticalPoint& cp : m.critical_points) {
            aid.push_back(cp.id);
            cell.push_back(cp.cell);
            index.push_back(cp.index);
            doubled.push_back(cp.doubled.x);
            doubled.push_back(cp.doubled.y);
            doubled.push_back(cp.doubled.z);
            midpoint.insert(midpoint.end(), cp.midpoint.begin(), cp.midpoint.end());
            value.push_back(cp.value);
        }
        std::vector<std::uint64_t> mult;
        for (const Arc& a : m.arcs) {
            src.push_back(a.src);
            dst.push_back(a.dst);
            mult.push_back(a.multiplicity);
        }
        b.put("cp_id", aid);
        b.put("cp_cell", cell);
        b.put("cp_index", index);
        b.put("cp_doubled", doubled);
        b.put("cp_midpoint", midpoint);
        b.put("cp_value", value);
        b.put("arc_src", src);
        b.put("arc_dst", dst);
        b.put("arc_mult", mult);
        b.put_scalar<std::uint64_t>("input_hash", m.input_hash);
        b.put_scalar<std::int64_t>("euler", m.euler());
        b.put("timings", std::vector<double>{t.gradient, t.critical, t.extrema, t.reachability,
                                             t.counting});
        b.put_scalar("wall", wall);
        b.put_scalar("hash_seconds", hash_secs);
        if (m.labels) {
            b.put("labels_min", m.labels->vertex_to_min);
            b.put("labels_max", m.labels->cube_to_max);
        }
        if (want_text) {
            const std::string js = serialize_json(m), c1 = critical_points_csv(m),
                              c2 = arcs_csv(m);
            b.put("json", std::vector<std::uint8_t>(js.begin(), js.end()));
            b.put("cp_csv", std::vector<std::uint8_t>(c1.begin(), c1.end()));
            b.put("arcs_csv", std::vector<std::uint8_t>(c2.begin(), c2.end()));
            if (m.labels) {
                const std::string l0 = label_volume_bytes(m.labels->vertex_to_min);
                b.put("labels_min_bytes", std::vector<std::uint8_t>(l0.begin(), l0.end()));
            }
            const BoundaryReport br = boundary_check(m);
            b.put_scalar<std::uint64_t>("boundary_odd_pairs", br.odd_pairs.size());
        }
    });
}

}  // extern "C"

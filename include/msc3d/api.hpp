// msc3d C++ drop-in API of the B200 build.
//
// Same namespace, type names, member names, function signatures, default arguments
// and exception types as the reference's public headers
// (/root/reference/proj/include/msc3d/{grid,gradient,extrema,saddle_graph,
// path_matrix,msc,volume,serialize}.hpp), so code written against the reference -
// including its unit tests - compiles unchanged against this header.  The per-name
// headers next to this file (msc3d/grid.hpp, ...) all forward here.
//
// Every pipeline stage is executed by the sm_100a kernels behind the C ABI in
// include/msc3d_cuda.h (paper_2009_03707_b200/csrc/msc3d_api.cpp does the
// marshalling); `threads` arguments are accepted for source compatibility and
// ignored (results never depend on them, as in the reference).  O(1) lattice
// queries (pack/unpack, facets, successors, compare_cells, ...) and host audits
// (validate_gradient, boundary_check, query_arcs) run on the host.
#pragma once

#include <array>
#include <compare>
#include <cstddef>
#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

namespace msc3d {

// ---------------------------------------------------------------- grid.hpp:33-149
using CellIndex = std::uint32_t;
using VertexIndex = std::uint32_t;

template <typename T, int N>
struct SmallList {
    std::array<T, N> item{};
    int count = 0;
    void push(T v) { item[static_cast<std::size_t>(count++)] = v; }
    const T* begin() const { return item.data(); }
    const T* end() const { return item.data() + count; }
    T operator[](int i) const { return item[static_cast<std::size_t>(i)]; }
};
using CellList = SmallList<CellIndex, 6>;
using VertexList = SmallList<VertexIndex, 8>;

struct GridDims {
    std::int64_t nx = 0, ny = 0, nz = 0;
    GridDims() = default;
    GridDims(std::int64_t nx_, std::int64_t ny_, std::int64_t nz_);  // invalid_argument
    std::int64_t ex() const { return 2 * nx - 1; }
    std::int64_t ey() const { return 2 * ny - 1; }
    std::int64_t ez() const { return 2 * nz - 1; }
    std::uint64_t vertex_count() const {
        return static_cast<std::uint64_t>(nx) * static_cast<std::uint64_t>(ny) * static_cast<std::uint64_t>(nz);
    }
    std::uint64_t cube_count() const {
        return static_cast<std::uint64_t>(nx - 1) * static_cast<std::uint64_t>(ny - 1) *
               static_cast<std::uint64_t>(nz - 1);
    }
    std::uint64_t total_cells() const {
        return static_cast<std::uint64_t>(ex()) * static_cast<std::uint64_t>(ey()) * static_cast<std::uint64_t>(ez());
    }
    bool operator==(const GridDims&) const = default;
};

struct CellCoord {
    std::int32_t x = 0, y = 0, z = 0;
    bool operator==(const CellCoord&) const = default;
};

CellIndex pack_cell(const GridDims& d, CellCoord c);
CellCoord unpack_cell(const GridDims& d, CellIndex id);
inline int cell_dimension(CellCoord c) { return (c.x & 1) + (c.y & 1) + (c.z & 1); }
int cell_dimension(const GridDims& d, CellIndex id);
CellList facets(const GridDims& d, CellIndex id);
CellList cofacets(const GridDims& d, CellIndex id);
VertexList cell_vertices(const GridDims& d, CellIndex id);
bool cell_on_boundary(const GridDims& d, CellIndex id);

struct ScalarField {
    GridDims dims;
    std::vector<double> values;
    ScalarField() = default;
    ScalarField(GridDims d, std::vector<double> v);  // invalid_argument: size / non-finite
    double operator[](VertexIndex v) const { return values[v]; }
};

struct CellOrderKey {
    std::array<double, 8> value{};
    std::array<VertexIndex, 8> vertex{};
    int count = 0;
};
CellOrderKey cell_order_key(const ScalarField& f, CellIndex id);
std::strong_ordering compare_keys(const CellOrderKey& a, const CellOrderKey& b);
std::strong_ordering compare_cells(const ScalarField& f, CellIndex a, CellIndex b);
VertexIndex max_vertex_of(const ScalarField& f, CellIndex id);

// ---------------------------------------------------------------- gradient.hpp:29-98
namespace pair_code {
constexpr std::uint8_t kUnset = 0;
constexpr std::uint8_t kCritical = 1;
constexpr std::uint8_t kFacetBase = 2;
constexpr std::uint8_t kCofacetBase = 8;
inline std::uint8_t with_facet(int axis, int sign) {
    return static_cast<std::uint8_t>(kFacetBase + axis * 2 + (sign > 0 ? 1 : 0));
}
inline std::uint8_t with_cofacet(int axis, int sign) {
    return static_cast<std::uint8_t>(kCofacetBase + axis * 2 + (sign > 0 ? 1 : 0));
}
}  // namespace pair_code

struct GradientField {
    GridDims dims;
    std::vector<std::uint8_t> code;
    bool is_critical(CellIndex c) const { return code[c] == pair_code::kCritical; }
    bool is_paired_with_facet(CellIndex c) const {
        return code[c] >= pair_code::kFacetBase && code[c] < pair_code::kCofacetBase;
    }
    bool is_paired_with_cofacet(CellIndex c) const { return code[c] >= pair_code::kCofacetBase; }
    CellIndex partner(CellIndex c) const {
        const std::uint8_t k = code[c];
        const int dir = k - (k < pair_code::kCofacetBase ? pair_code::kFacetBase : pair_code::kCofacetBase);
        const std::int64_t step = (dir >> 1) == 0 ? 1 : ((dir >> 1) == 1 ? dims.ex() : dims.ex() * dims.ey());
        return static_cast<CellIndex>(static_cast<std::int64_t>(c) + ((dir & 1) ? step : -step));
    }
};

GradientField assign_gradient(const ScalarField& f, int threads = 0);

struct CriticalCells {
    std::vector<CellIndex> by_dim[4];
    std::int64_t euler() const {
        return static_cast<std::int64_t>(by_dim[0].size()) - static_cast<std::int64_t>(by_dim[1].size()) +
               static_cast<std::int64_t>(by_dim[2].size()) - static_cast<std::int64_t>(by_dim[3].size());
    }
};
CriticalCells extract_critical_cells(const GradientField& g, int threads = 0);

struct GradientReport {
    std::uint64_t matching_violations = 0;
    std::uint64_t cells_in_closed_vpath = 0;
    bool acyclicity_checked = false;
    bool degenerate = false;
    std::vector<CellIndex> samples;
    bool ok() const { return matching_violations == 0 && cells_in_closed_vpath == 0; }
};
GradientReport validate_gradient(const GradientField& g, std::uint64_t max_cells_for_cycles = 100000);

// ---------------------------------------------------------------- extrema.hpp:27-78
std::uint64_t dense_cell_count(const GridDims& d, int dim);
CellIndex dense_to_cell(const GridDims& d, int dim, std::uint32_t i);
std::uint32_t cell_to_dense(const GridDims& d, int dim, CellIndex c);

struct ParentForest {
    GridDims dims;
    int dim = 0;
    std::vector<std::uint32_t> parent;
};
ParentForest build_forest(const GradientField& g, int dim, int threads = 0);

struct RootLabels {
    std::vector<std::uint32_t> label;
    int rounds = 0;
};
RootLabels find_roots(const ParentForest& forest, int threads = 0);

struct SaddleExtremumArc {
    CellIndex saddle = 0;
    CellIndex extremum = 0;
    std::uint32_t multiplicity = 0;
    bool operator==(const SaddleExtremumArc&) const = default;
};
std::vector<SaddleExtremumArc> saddle_extremum_arcs(const GradientField& g, const RootLabels& labels0,
                                                    const RootLabels& labels3, int threads = 0);

struct Segmentation {
    GridDims dims;
    std::vector<std::uint32_t> vertex_to_min;
    std::vector<std::uint32_t> cube_to_max;
};
Segmentation extremum_segmentation(const GridDims& dims, const RootLabels& labels0, const RootLabels& labels3);

// ---------------------------------------------------------------- saddle_graph.hpp:27-74
struct DagSuccessor {
    enum Kind : std::uint8_t { kEdge, kTerminal2Saddle };
    Kind kind = kEdge;
    CellIndex cell = 0;
    bool operator==(const DagSuccessor&) const = default;
};
using SuccessorList = SmallList<DagSuccessor, 4>;
SuccessorList successors(const GradientField& g, CellIndex e);

struct MarkedSubgraph {
    GridDims dims;
    std::vector<std::uint8_t> marked;
    std::vector<CellIndex> one_saddles;
    std::vector<CellIndex> two_saddles;
};
MarkedSubgraph mark_reachable(const GradientField& g, const std::vector<CellIndex>& one_saddles,
                              int threads = 0);

struct MinorEdge {
    std::uint32_t src = 0;
    std::uint32_t dst = 0;
    std::uint64_t multiplicity = 0;
    bool operator==(const MinorEdge&) const = default;
};
struct DagMinor {
    std::vector<CellIndex> one_saddles;
    std::vector<CellIndex> junctions;
    std::vector<CellIndex> two_saddles;
    std::vector<MinorEdge> s1_to_j, j_to_j, j_to_s2, s1_to_s2;
};
DagMinor build_minor(const MarkedSubgraph& m, const GradientField& g, int threads = 0);

// ---------------------------------------------------------------- path_matrix.hpp:27-64
struct SparseCountMatrix {
    std::uint32_t rows = 0, cols = 0;
    std::vector<std::uint64_t> row_ptr;
    std::vector<std::uint32_t> col_idx;
    std::vector<std::uint64_t> count;
    std::uint64_t nnz() const { return col_idx.size(); }
    bool operator==(const SparseCountMatrix&) const = default;
};
SparseCountMatrix from_edges(const std::vector<MinorEdge>& edges, std::uint32_t rows, std::uint32_t cols);
SparseCountMatrix sp_multiply(const SparseCountMatrix& x, const SparseCountMatrix& y, int threads = 0);
SparseCountMatrix sp_add(const SparseCountMatrix& x, const SparseCountMatrix& y, int threads = 0);

struct SaddleConnection {
    CellIndex one_saddle = 0;
    CellIndex two_saddle = 0;
    std::uint64_t paths = 0;
    bool operator==(const SaddleConnection&) const = default;
};
std::vector<SaddleConnection> count_paths(const DagMinor& minor, int threads = 0);

// ---------------------------------------------------------------- msc.hpp:24-105
struct CriticalPoint {
    std::uint32_t id = 0;
    CellIndex cell = 0;
    int index = 0;
    CellCoord doubled;
    std::array<double, 3> midpoint{};
    double value = 0;
    bool operator==(const CriticalPoint&) const = default;
};
struct Arc {
    std::uint32_t src = 0;
    std::uint32_t dst = 0;
    std::uint64_t multiplicity = 0;
    bool operator==(const Arc&) const = default;
};
struct LabelVolumes {
    static constexpr std::uint32_t kNoLabel = 0xffffffffu;
    std::vector<std::uint32_t> vertex_to_min;
    std::vector<std::uint32_t> cube_to_max;
    bool operator==(const LabelVolumes&) const = default;
};
struct MSComplex {
    GridDims dims;
    std::string dtype = "f64";
    std::uint64_t input_hash = 0;
    std::string tie_break = "vertex-index-v1";
    std::vector<CriticalPoint> critical_points;
    std::vector<Arc> arcs;
    std::optional<LabelVolumes> labels;
    std::uint64_t count_by_index(int index) const;
    std::int64_t euler() const;
    bool operator==(const MSComplex&) const = default;
};
struct StageTimings {
    double gradient = 0;
    double critical = 0;
    double extrema = 0;
    double reachability = 0;
    double counting = 0;
};
struct ComputeOptions {
    int threads = 0;
    bool with_segmentation = false;
    bool validate = false;
    std::string source_dtype = "f64";
    StageTimings* timings = nullptr;  // device seconds per stage
};
MSComplex compute(const ScalarField& f, const ComputeOptions& opt = {});
std::uint64_t field_hash(const ScalarField& f);

struct BoundaryReport {
    std::vector<std::array<std::uint32_t, 2>> odd_pairs;
    bool ok() const { return odd_pairs.empty(); }
};
BoundaryReport boundary_check(const MSComplex& m);
std::vector<Arc> query_arcs(const MSComplex& m, std::uint32_t cp_id);

// ---------------------------------------------------------------- volume.hpp:20-57
class IoError : public std::runtime_error {
  public:
    using std::runtime_error::runtime_error;
};
enum class SampleType : std::uint8_t { u8, u16, f32, f64 };
SampleType parse_sample_type(const std::string& name);
const char* sample_type_name(SampleType t);
std::size_t sample_size(SampleType t);
struct VolumeSpec {
    std::string path;
    GridDims dims;
    SampleType dtype = SampleType::f64;
    bool big_endian = false;
};
ScalarField read_volume(const VolumeSpec& spec);
// Extension (not in the reference API): compute(read_volume(spec), opt) with the same
// results and errors; f32 little-endian files are read straight into pinned upload
// memory (no vector of doubles).  The CLI's path.
MSComplex compute_volume(const VolumeSpec& spec, const ComputeOptions& opt = {});

// ---------------------------------------------------------------- serialize.hpp:21-45
class ParseError : public std::runtime_error {
  public:
    ParseError(const std::string& what, std::size_t offset) : std::runtime_error(what), byte_offset(offset) {}
    std::size_t byte_offset = 0;
};
std::string serialize_json(const MSComplex& m);
MSComplex deserialize_json(std::string_view bytes);
std::string critical_points_csv(const MSComplex& m);
std::string arcs_csv(const MSComplex& m);
std::string label_volume_bytes(const std::vector<std::uint32_t>& labels);

}  // namespace msc3d

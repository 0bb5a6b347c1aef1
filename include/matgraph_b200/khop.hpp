// matgraph_b200: the C++ drop-in for the reference's k-hop count path.
//
// Signature-compatible with the reference (namespace matgraph) for every
// symbol on the path, so a caller of
//   proj/core/include/matgraph/execute.hpp:52-68  (KHopQuery, k_hop_frontier, k_hop_count)
//   proj/core/include/matgraph/graph.hpp:20-124   (RelationRef, PropertyGraph load API)
//   proj/core/include/matgraph/bench.hpp:16-156   (RMAT, build_bench_graph, pick_seeds,
//                                                  summarize, run_khop_benchmark, CSV)
//   proj/core/include/matgraph/error.hpp:10-66    (Error, ContractError, HarnessError)
// compiles against this header with the same signatures (mangled names
// included) for every symbol it declares. The traversal runs on a B200
// through the C ABI of include/mgk.h; the relation matrix is uploaded once per
// (relation, flush state) and cached like the reference caches its transpose
// (graph.cpp:90-102). Labels and properties are accepted and stored (the
// k-hop path never reads them). Not provided: the Cypher frontend / planner /
// executor, the server, snapshots. BfsOracle (bench.hpp:73-91) is declared
// here but defined only by the test infrastructure (oracle/dropin_bfs.cpp),
// which the drop-in's test binaries link; the product library has no oracle.
#pragma once

#include <cstdint>
#include <filesystem>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <tuple>
#include <variant>
#include <vector>

struct mgk_graph;

namespace matgraph {

// ---- errors (error.hpp:10-66) ----------------------------------------------------
class Error : public std::runtime_error {
public:
    explicit Error(const std::string& message) : std::runtime_error(message) {}
};
class ContractError : public Error {
    using Error::Error;
};
class HarnessError : public Error {
    using Error::Error;
};

inline constexpr std::uint32_t kMaxHops = 32;  // ast.hpp:15

enum class TraverseMode : std::uint8_t { Exact, Cumulative };  // plan.hpp:17

// ---- semirings (sparse.hpp:45-67) -------------------------------------------------
enum class BinaryOp : std::uint8_t { BoolOr, BoolAnd, Plus, Times, Min };
std::int64_t apply(BinaryOp op, std::int64_t lhs, std::int64_t rhs);
struct Semiring {
    BinaryOp add_op = BinaryOp::BoolOr;
    BinaryOp mul_op = BinaryOp::BoolAnd;
    std::int64_t add_identity = 0;
    static const Semiring& bool_or_and();
    static const Semiring& plus_times();
    static const Semiring& min_plus();
    bool is_boolean() const noexcept { return add_op == BinaryOp::BoolOr; }
    friend bool operator==(const Semiring&, const Semiring&) = default;
};

struct MatrixTuple {  // sparse.hpp:69-75
    std::uint64_t row = 0;
    std::uint64_t col = 0;
    std::int64_t value = 1;
    friend bool operator==(const MatrixTuple&, const MatrixTuple&) = default;
};

// ---- sparse types (sparse.hpp:13-43, 83-134), the subset the path reads -----------
class BitVector {
public:
    BitVector() = default;
    explicit BitVector(std::uint64_t dimension) : dimension_(dimension) {}
    static BitVector from_sorted(std::uint64_t dimension, std::vector<std::uint64_t> indices);
    std::uint64_t dimension() const noexcept { return dimension_; }
    std::uint64_t nvals() const noexcept { return indices_.size(); }
    bool empty() const noexcept { return indices_.empty(); }
    std::span<const std::uint64_t> indices() const noexcept { return indices_; }
    friend bool operator==(const BitVector&, const BitVector&) = default;

private:
    std::uint64_t dimension_ = 0;
    std::vector<std::uint64_t> indices_;
};

class SparseMatrix {
public:
    SparseMatrix() = default;
    SparseMatrix(std::uint64_t nrows, std::uint64_t ncols)
        : nrows_(nrows), ncols_(ncols), row_ptr_(nrows + 1, 0) {}
    /// Valued when `vals` is non-empty (one int64 per entry), like the reference.
    static SparseMatrix from_parts(std::uint64_t nrows, std::uint64_t ncols,
                                   std::vector<std::uint64_t> row_ptr,
                                   std::vector<std::uint64_t> col_idx,
                                   std::vector<std::int64_t> vals = {});
    std::uint64_t nrows() const noexcept { return nrows_; }
    std::uint64_t ncols() const noexcept { return ncols_; }
    std::uint64_t nvals() const noexcept { return col_idx_.size(); }
    bool has_values() const noexcept { return valued_; }
    bool valued() const noexcept { return valued_; }
    std::span<const std::uint64_t> row_ptr() const noexcept { return row_ptr_; }
    std::span<const std::uint64_t> col_idx() const noexcept { return col_idx_; }
    std::span<const std::int64_t> values() const noexcept { return vals_; }
    std::span<const std::uint64_t> row(std::uint64_t r) const;
    std::span<const std::int64_t> row_values(std::uint64_t r) const;
    bool contains(std::uint64_t r, std::uint64_t c) const;
    /// (row, col, value) in row-major order; value 1 for a structural matrix.
    std::vector<MatrixTuple> extract_tuples() const;

private:
    std::uint64_t nrows_ = 0, ncols_ = 0;
    bool valued_ = false;
    std::vector<std::uint64_t> row_ptr_ = {0};
    std::vector<std::uint64_t> col_idx_;
    std::vector<std::int64_t> vals_;
};

std::uint64_t nvals(const SparseMatrix& m);
std::uint64_t nvals(const BitVector& v);

/// mxm (sparse.cpp:292-363) computed on the GPU (mgk_mxm): C = A (+.*) B,
/// restricted to the pattern of `mask` when given. Same results and messages
/// as the reference ("mxm: inner dimensions disagree ...", "mxm: mask shape ...").
SparseMatrix mxm(const SparseMatrix& a, const SparseMatrix& b,
                 const Semiring& semiring = Semiring::bool_or_and(), const SparseMatrix* mask = nullptr);

// ---- property values (value.hpp:10-46) ---------------------------------------------
/// Int / float / bool / string; `Value("x")` is a string (no decay to bool).
class Value {
public:
    enum class Type { Int, Float, Bool, String };
    Value() : v_(std::int64_t{0}) {}
    Value(std::int64_t i) : v_(i) {}
    Value(int i) : v_(std::int64_t{i}) {}
    Value(double d) : v_(d) {}
    Value(bool b) : v_(b) {}
    Value(std::string s) : v_(std::move(s)) {}
    Value(std::string_view s) : v_(std::string(s)) {}
    Value(const char* s) : v_(std::string(s)) {}
    Type type() const noexcept { return static_cast<Type>(v_.index()); }
    bool is_int() const noexcept { return type() == Type::Int; }
    bool is_float() const noexcept { return type() == Type::Float; }
    bool is_bool() const noexcept { return type() == Type::Bool; }
    bool is_string() const noexcept { return type() == Type::String; }
    bool is_numeric() const noexcept { return is_int() || is_float(); }
    std::int64_t as_int() const { return std::get<std::int64_t>(v_); }
    double as_float() const { return std::get<double>(v_); }
    bool as_bool() const { return std::get<bool>(v_); }
    const std::string& as_string() const { return std::get<std::string>(v_); }
    friend bool operator==(const Value&, const Value&) = default;

private:
    std::variant<std::int64_t, double, bool, std::string> v_;
};
using PropertyMap = std::map<std::string, Value>;

// ---- graph store (graph.hpp:20-124), load API + matrix access ---------------------
struct RelationRef {
    std::optional<std::string> name;  // nullopt = ANY
    RelationRef() = default;
    RelationRef(std::string n) : name(std::move(n)) {}
    RelationRef(std::string_view n) : name(std::string(n)) {}
    RelationRef(const char* n) : name(std::string(n)) {}
    static RelationRef any() { return {}; }
    bool is_any() const noexcept { return !name.has_value(); }
    friend bool operator==(const RelationRef&, const RelationRef&) = default;
};

// A relation matrix resident on one GPU (owning handle of the C ABI graph).
class DeviceMatrix {
public:
    explicit DeviceMatrix(mgk_graph* h) : h_(h) {}
    ~DeviceMatrix();
    DeviceMatrix(const DeviceMatrix&) = delete;
    DeviceMatrix& operator=(const DeviceMatrix&) = delete;
    mgk_graph* handle() const noexcept { return h_; }

private:
    mgk_graph* h_;
};

class PropertyGraph {
public:
    explicit PropertyGraph(std::uint64_t initial_capacity = 16);
    PropertyGraph(PropertyGraph&&) noexcept = default;
    PropertyGraph& operator=(PropertyGraph&&) noexcept = default;
    PropertyGraph(const PropertyGraph&) = delete;
    PropertyGraph& operator=(const PropertyGraph&) = delete;

    /// Allocates the next node id (graph.cpp:31-52: labels must be identifiers).
    std::uint64_t create_node(const std::vector<std::string>& labels, PropertyMap props = {});
    /// Records a directed typed edge (graph.cpp:54-82 contract and messages);
    /// re-creating an edge overwrites its properties.
    void create_edge(std::uint64_t src, const std::string& relation, std::uint64_t dst,
                     PropertyMap props = {});
    const PropertyMap& node_props(std::uint64_t id) const;
    const PropertyMap* edge_props(std::uint64_t src, std::string_view relation, std::uint64_t dst) const;
    /// Sorted labels of one node.
    std::vector<std::string> node_labels(std::uint64_t id) const;

    std::uint64_t node_count() const noexcept { return node_count_; }
    std::uint64_t capacity() const noexcept { return capacity_; }

    /// Flushes pending edges; unknown names yield the empty matrix (graph.cpp:84-88).
    const SparseMatrix& relation_matrix(const RelationRef& rel = RelationRef::any()) const;
    /// Transposed adjacency (graph.cpp:90-102): computed lazily on the host,
    /// mutex-guarded, cached until the next write.
    const SparseMatrix& transposed_matrix(const RelationRef& rel = RelationRef::any()) const;
    /// The matrix on `device` (uploaded on first use, cached until the next
    /// flush that changes it; mutex-guarded like transposed_matrix).
    const DeviceMatrix& device_matrix(const RelationRef& rel = RelationRef::any(),
                                      int device = 0) const;
    std::vector<std::string> relation_names() const;
    /// Sort + dedup pending pairs into the CSR of each relation and ANY
    /// (graph.cpp:167-215); drops device caches of changed matrices.
    void flush() const;

private:
    struct Slot {
        SparseMatrix matrix;
        std::vector<std::pair<std::uint64_t, std::uint64_t>> pending;
        std::map<int, std::shared_ptr<DeviceMatrix>> device;
        std::optional<SparseMatrix> transposed;
    };
    void grow_to(std::uint64_t needed);
    const Slot* find_slot(const RelationRef& rel) const;
    static void flush_slot(Slot& slot, std::uint64_t dim);

    std::uint64_t capacity_ = 0;
    std::uint64_t node_count_ = 0;
    mutable std::map<std::string, Slot, std::less<>> relations_;
    mutable Slot any_;
    mutable Slot empty_;
    mutable std::unique_ptr<std::mutex> device_mutex_;
    std::map<std::string, std::vector<std::uint64_t>, std::less<>> labels_;
    std::vector<PropertyMap> node_props_;
    std::map<std::tuple<std::uint64_t, std::string, std::uint64_t>, PropertyMap> edge_props_;
};

// ---- the k-hop kernel (execute.hpp:52-68) ------------------------------------------
struct KHopQuery {
    std::uint64_t seed = 0;
    std::uint32_t k = 1;
    RelationRef relation = RelationRef::any();
    TraverseMode mode = TraverseMode::Exact;
};

/// Masked BFS from the seed (execute.cpp:347-371), on the GPU.
BitVector k_hop_frontier(const PropertyGraph& graph, const KHopQuery& query);
/// nvals(k_hop_frontier(graph, query)) (execute.cpp:373-375), on the GPU.
std::uint64_t k_hop_count(const PropertyGraph& graph, const KHopQuery& query);
/// Additive API: one k_hop_count per seed in one device call (bit-exact per seed).
std::vector<std::uint64_t> k_hop_count_batch(const PropertyGraph& graph,
                                             std::span<const std::uint64_t> seeds, std::uint32_t k,
                                             const RelationRef& relation = RelationRef::any(),
                                             TraverseMode mode = TraverseMode::Exact);

/// walk_targets (execute.cpp:43-60): sorted ids whose shortest nonempty walk
/// from `src` has length in [min, max] (visited starts empty, so `src` itself
/// appears on a cycle) — the VarLenTraverse step of MATCH (a)-[*min..max]->(b).
std::vector<std::uint64_t> walk_targets(const PropertyGraph& graph, std::uint64_t src,
                                        std::uint32_t min, std::uint32_t max,
                                        const RelationRef& relation = RelationRef::any());
/// |walk_targets| for many sources in one device call.
std::vector<std::uint64_t> walk_count_batch(const PropertyGraph& graph,
                                            std::span<const std::uint64_t> sources, std::uint32_t min,
                                            std::uint32_t max,
                                            const RelationRef& relation = RelationRef::any());

// ---- benchmark harness (bench.hpp:16-156) -------------------------------------------
struct RmatParams {
    std::uint32_t scale = 14;
    std::uint32_t edge_factor = 16;
    double a = 0.57, b = 0.19, c = 0.19, d = 0.05;
    std::uint64_t rng_seed = 1;
    std::uint64_t node_count() const noexcept { return std::uint64_t{1} << scale; }
    std::uint64_t edge_count() const noexcept { return std::uint64_t{edge_factor} << scale; }
    void validate() const;
};

struct EdgeTuple {
    std::uint32_t src = 0;
    std::uint32_t dst = 0;
    friend bool operator==(const EdgeTuple&, const EdgeTuple&) = default;
};
using EdgeList = std::vector<EdgeTuple>;

inline constexpr std::string_view kBenchRelation = "EDGE";

EdgeList rmat_generate(const RmatParams& params);
/// bench.cpp:139-173: `src<TAB>dst` lines, HarnessError with the line number.
EdgeList load_edge_list(const std::filesystem::path& path);
/// max endpoint + 1, 0 for an empty list (bench.cpp:175-183).
std::uint64_t edge_list_node_count(const EdgeList& edges);
PropertyGraph build_bench_graph(const EdgeList& edges, std::uint64_t node_count);
std::vector<std::uint64_t> pick_seeds(const PropertyGraph& graph, std::size_t n,
                                      std::uint64_t rng_seed);

/// Queue-based BFS oracle over a raw edge list (bench.hpp:73-91). DECLARED
/// ONLY: the definition is test infrastructure (oracle/dropin_bfs.cpp over the
/// C oracle), linked into test binaries, never into libmatgraph_b200.so.
class BfsOracle {
public:
    BfsOracle(const EdgeList& edges, std::uint64_t node_count);
    ~BfsOracle();
    BfsOracle(BfsOracle&&) noexcept;
    BfsOracle& operator=(BfsOracle&&) noexcept;
    std::uint64_t count(std::uint64_t seed, std::uint32_t k, TraverseMode mode) const;
    std::uint64_t node_count() const noexcept { return node_count_; }

private:
    void* impl_ = nullptr;
    std::uint64_t node_count_ = 0;
};
std::uint64_t bfs_oracle(const PropertyGraph& graph, std::uint64_t seed, std::uint32_t k, TraverseMode mode);

struct SeedRun {
    std::uint64_t seed = 0;
    std::uint64_t count = 0;
    std::int64_t elapsed_us = 0;
};
struct SectionStats {
    double mean_us = 0.0, median_us = 0.0, p99_us = 0.0, mean_count = 0.0;
};
SectionStats summarize(const std::vector<SeedRun>& runs);
struct KHopSection {
    std::uint32_t k = 0;
    std::vector<SeedRun> runs;
    SectionStats stats;
};
struct KHopReport {
    TraverseMode mode = TraverseMode::Exact;
    std::vector<KHopSection> sections;
};
struct BenchSchedule {
    std::vector<std::uint32_t> ks;
    std::vector<std::size_t> seeds_per_k;
    TraverseMode mode = TraverseMode::Exact;
    std::uint64_t rng_seed = 1;
    void validate() const;
};
/// bench.cpp:311-343: sequential per-query timing like the reference.
KHopReport run_khop_benchmark(const PropertyGraph& graph, const BenchSchedule& schedule);
/// Additive overload: batched = true issues one device call per section and
/// spreads its wall time over the section's seeds.
KHopReport run_khop_benchmark(const PropertyGraph& graph, const BenchSchedule& schedule, bool batched);
std::string report_csv_string(const KHopReport& report);
void report_csv(const KHopReport& report, const std::filesystem::path& path);

}  // namespace matgraph

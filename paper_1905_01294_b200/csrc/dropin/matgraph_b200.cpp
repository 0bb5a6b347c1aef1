// matgraph_b200: the C++ drop-in for the reference's k-hop path (see
// include/matgraph_b200/khop.hpp). Host logic mirrors the reference's
// contracts and messages; every traversal goes through the C ABI (mgk.h).
#include "matgraph_b200/khop.hpp"

#include <algorithm>
#include <charconv>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <limits>
#include <random>
#include <string>

#include "mgk.h"

namespace matgraph {

namespace {

template <typename... A>
std::string fmt(const char* f, A... a) {
    char buf[512];
    std::snprintf(buf, sizeof buf, f, a...);
    return buf;
}

[[noreturn]] void throw_mgk(int rc) {
    const std::string msg = mgk_last_error();
    if (rc == MGK_ECONTRACT || rc == MGK_ERANGE) throw ContractError(msg);
    if (rc == MGK_EHARNESS) throw HarnessError(msg);
    throw Error(msg);
}

bool is_identifier(std::string_view name) {  // encoding.cpp:111-119
    if (name.empty()) return false;
    auto head = [](char c) { return (c >= 'A' && c <= 'Z') || (c >= 'a' && c <= 'z') || c == '_'; };
    if (!head(name[0])) return false;
    for (char c : name.substr(1))
        if (!head(c) && !(c >= '0' && c <= '9')) return false;
    return true;
}

std::string format_double(double value) {  // encoding.cpp:67-72
    char buf[64];
    auto [end, ec] = std::to_chars(buf, buf + sizeof(buf), value);
    if (ec != std::errc{}) throw Error("failed to format double");
    return std::string(buf, end);
}

constexpr std::uint64_t kMinCapacity = 16;

// bench.cpp:37-48
double unit_double(std::mt19937_64& rng) { return static_cast<double>(rng() >> 11) * 0x1.0p-53; }
std::uint64_t bounded_draw(std::mt19937_64& rng, std::uint64_t bound) {
    const std::uint64_t max = std::numeric_limits<std::uint64_t>::max();
    const std::uint64_t limit = max - max % bound;
    std::uint64_t draw = rng();
    while (draw >= limit) draw = rng();
    return draw % bound;
}

}  // namespace

// ---- sparse types --------------------------------------------------------------------
BitVector BitVector::from_sorted(std::uint64_t dimension, std::vector<std::uint64_t> indices) {
    for (std::size_t i = 0; i < indices.size(); ++i) {
        if (indices[i] >= dimension)
            throw Error(fmt("BitVector invariant violated: index %llu >= dimension %llu",
                            (unsigned long long)indices[i], (unsigned long long)dimension));
        if (i > 0 && indices[i - 1] >= indices[i])
            throw Error(fmt("BitVector invariant violated: indices not strictly increasing at %zu", i));
    }
    BitVector v(dimension);
    v.indices_ = std::move(indices);
    return v;
}

SparseMatrix SparseMatrix::from_parts(std::uint64_t nrows, std::uint64_t ncols,
                                      std::vector<std::uint64_t> row_ptr,
                                      std::vector<std::uint64_t> col_idx,
                                      std::vector<std::int64_t> vals) {
    if (row_ptr.size() != nrows + 1 || row_ptr.front() != 0 || row_ptr.back() != col_idx.size())
        throw Error("SparseMatrix invariant violated: row_ptr shape");
    if (!vals.empty() && vals.size() != col_idx.size())
        throw Error("SparseMatrix invariant violated: value count");
    SparseMatrix m;
    m.nrows_ = nrows;
    m.ncols_ = ncols;
    m.valued_ = !vals.empty();
    m.row_ptr_ = std::move(row_ptr);
    m.col_idx_ = std::move(col_idx);
    m.vals_ = std::move(vals);
    return m;
}

std::span<const std::int64_t> SparseMatrix::row_values(std::uint64_t r) const {
    if (r >= nrows_)
        throw ContractError(fmt("row %llu out of range for %llux%llu matrix", (unsigned long long)r,
                                (unsigned long long)nrows_, (unsigned long long)ncols_));
    if (!valued_) return {};
    return std::span(vals_).subspan(row_ptr_[r], row_ptr_[r + 1] - row_ptr_[r]);
}

bool SparseMatrix::contains(std::uint64_t r, std::uint64_t c) const {
    const auto cols = row(r);
    return std::binary_search(cols.begin(), cols.end(), c);
}

std::vector<MatrixTuple> SparseMatrix::extract_tuples() const {
    std::vector<MatrixTuple> out;
    out.reserve(col_idx_.size());
    for (std::uint64_t r = 0; r < nrows_; ++r)
        for (std::uint64_t p = row_ptr_[r]; p < row_ptr_[r + 1]; ++p)
            out.push_back({r, col_idx_[p], valued_ ? vals_[p] : 1});
    return out;
}

// ---- semirings (sparse.cpp:69-93) --------------------------------------------------
std::int64_t apply(BinaryOp op, std::int64_t lhs, std::int64_t rhs) {
    switch (op) {
        case BinaryOp::BoolOr: return (lhs != 0 || rhs != 0) ? 1 : 0;
        case BinaryOp::BoolAnd: return (lhs != 0 && rhs != 0) ? 1 : 0;
        case BinaryOp::Plus: return (std::int64_t)((std::uint64_t)lhs + (std::uint64_t)rhs);
        case BinaryOp::Times: return (std::int64_t)((std::uint64_t)lhs * (std::uint64_t)rhs);
        case BinaryOp::Min: return lhs < rhs ? lhs : rhs;
    }
    throw ContractError("unknown binary operator");
}

const Semiring& Semiring::bool_or_and() {
    static const Semiring s{BinaryOp::BoolOr, BinaryOp::BoolAnd, 0};
    return s;
}
const Semiring& Semiring::plus_times() {
    static const Semiring s{BinaryOp::Plus, BinaryOp::Times, 0};
    return s;
}
const Semiring& Semiring::min_plus() {
    static const Semiring s{BinaryOp::Min, BinaryOp::Plus, INT64_MAX};
    return s;
}

SparseMatrix mxm(const SparseMatrix& a, const SparseMatrix& b, const Semiring& semiring,
                 const SparseMatrix* mask) {
    int code = -1;
    if (semiring == Semiring::bool_or_and()) code = MGK_SEMIRING_BOOL_OR_AND;
    else if (semiring == Semiring::plus_times()) code = MGK_SEMIRING_PLUS_TIMES;
    else if (semiring == Semiring::min_plus()) code = MGK_SEMIRING_MIN_PLUS;
    if (code < 0) throw ContractError("mxm: unsupported semiring");
    const std::uint64_t zero = 0;
    auto ci = [&](const SparseMatrix& m) { return m.nvals() ? m.col_idx().data() : &zero; };
    auto vals = [&](const SparseMatrix& m) -> const std::int64_t* {
        return m.valued() && m.nvals() ? m.values().data() : nullptr;
    };
    mgk_matrix* h = nullptr;
    const int rc = mgk_mxm(0, a.nrows(), a.ncols(), a.row_ptr().data(), ci(a), vals(a), b.nrows(), b.ncols(),
                           b.row_ptr().data(), ci(b), vals(b), code, mask ? mask->nrows() : 0,
                           mask ? mask->ncols() : 0, mask ? mask->row_ptr().data() : nullptr,
                           mask ? ci(*mask) : nullptr, &h);
    if (rc == MGK_ECONTRACT || rc == MGK_ERANGE) throw ContractError(mgk_last_error());
    if (rc) throw Error(mgk_last_error());
    std::uint64_t nr = 0, nc = 0, nnz = 0;
    int valued = 0;
    mgk_matrix_info(h, &nr, &nc, &nnz, &valued);
    std::vector<std::uint64_t> rp(nr + 1), c(nnz);
    std::vector<std::int64_t> v(valued ? nnz : 0);
    mgk_matrix_download(h, rp.data(), c.data(), valued ? v.data() : nullptr);
    mgk_matrix_free(h);
    return SparseMatrix::from_parts(nr, nc, std::move(rp), std::move(c), std::move(v));
}

std::span<const std::uint64_t> SparseMatrix::row(std::uint64_t r) const {
    if (r >= nrows_)
        throw ContractError(fmt("row %llu out of range for %llux%llu matrix", (unsigned long long)r,
                                (unsigned long long)nrows_, (unsigned long long)ncols_));
    return std::span(col_idx_).subspan(row_ptr_[r], row_ptr_[r + 1] - row_ptr_[r]);
}

std::uint64_t nvals(const SparseMatrix& m) { return m.nvals(); }
std::uint64_t nvals(const BitVector& v) { return v.nvals(); }

// ---- graph store ---------------------------------------------------------------------------
DeviceMatrix::~DeviceMatrix() {
    if (h_) mgk_graph_free(h_);
}

PropertyGraph::PropertyGraph(std::uint64_t initial_capacity)
    : capacity_(std::max(initial_capacity, kMinCapacity)),
      device_mutex_(std::make_unique<std::mutex>()) {
    any_.matrix = SparseMatrix(capacity_, capacity_);
    empty_.matrix = SparseMatrix(capacity_, capacity_);
}

void PropertyGraph::grow_to(std::uint64_t needed) {  // graph.cpp:236-248 (capacity doubling)
    if (needed <= capacity_) return;
    std::uint64_t cap = std::max(capacity_, kMinCapacity);
    while (cap < needed) cap *= 2;
    flush();
    auto pad = [cap](Slot& s) {
        std::vector<std::uint64_t> rp(s.matrix.row_ptr().begin(), s.matrix.row_ptr().end());
        rp.resize(cap + 1, rp.back());
        std::vector<std::uint64_t> ci(s.matrix.col_idx().begin(), s.matrix.col_idx().end());
        s.matrix = SparseMatrix::from_parts(cap, cap, std::move(rp), std::move(ci));
        s.device.clear();
        s.transposed.reset();
    };
    for (auto& [name, slot] : relations_) {
        (void)name;
        pad(slot);
    }
    pad(any_);
    empty_.matrix = SparseMatrix(cap, cap);
    empty_.device.clear();
    capacity_ = cap;
}

std::uint64_t PropertyGraph::create_node(const std::vector<std::string>& labels, PropertyMap props) {
    for (const auto& label : labels)  // graph.cpp:31-52
        if (!is_identifier(label))
            throw ContractError(fmt("label '%s' is not a valid identifier", label.c_str()));
    for (const auto& kv : props)
        if (!is_identifier(kv.first))
            throw ContractError(fmt("property key '%s' is not a valid identifier", kv.first.c_str()));
    grow_to(node_count_ + 1);
    const std::uint64_t id = node_count_++;
    for (const auto& label : labels) {
        auto& members = labels_[label];
        if (members.empty() || members.back() != id) members.push_back(id);  // ids ascend
    }
    node_props_.push_back(std::move(props));
    return id;
}

void PropertyGraph::create_edge(std::uint64_t src, const std::string& relation, std::uint64_t dst,
                                PropertyMap props) {
    if (src >= node_count_ || dst >= node_count_)  // graph.cpp:56-60
        throw ContractError(fmt("unknown node id %llu in edge (%llu)-[:%s]->(%llu)",
                                (unsigned long long)(src >= node_count_ ? src : dst),
                                (unsigned long long)src, relation.c_str(), (unsigned long long)dst));
    if (!is_identifier(relation))
        throw ContractError(fmt("relation type '%s' is not a valid identifier", relation.c_str()));
    for (const auto& kv : props)
        if (!is_identifier(kv.first))
            throw ContractError(fmt("property key '%s' is not a valid identifier", kv.first.c_str()));
    auto [it, inserted] = relations_.try_emplace(relation);
    if (inserted) it->second.matrix = SparseMatrix(capacity_, capacity_);
    it->second.pending.emplace_back(src, dst);
    any_.pending.emplace_back(src, dst);
    auto key = std::make_tuple(src, relation, dst);
    if (props.empty())
        edge_props_.erase(key);  // re-creating an edge overwrites its properties
    else
        edge_props_[key] = std::move(props);
}

const PropertyMap& PropertyGraph::node_props(std::uint64_t id) const {
    if (id >= node_count_) throw ContractError(fmt("unknown node id %llu", (unsigned long long)id));
    return node_props_[id];
}

const PropertyMap* PropertyGraph::edge_props(std::uint64_t src, std::string_view relation, std::uint64_t dst) const {
    auto it = edge_props_.find(std::make_tuple(src, std::string(relation), dst));
    return it == edge_props_.end() ? nullptr : &it->second;
}

std::vector<std::string> PropertyGraph::node_labels(std::uint64_t id) const {
    std::vector<std::string> out;
    for (const auto& [label, members] : labels_)  // map order: sorted by name
        if (std::binary_search(members.begin(), members.end(), id)) out.push_back(label);
    return out;
}

void PropertyGraph::flush_slot(Slot& slot, std::uint64_t dim) {  // graph.cpp:182-215
    if (slot.pending.empty()) return;
    auto& pending = slot.pending;
    for (std::uint64_t r = 0; r < slot.matrix.nrows(); ++r)
        for (std::uint64_t c : slot.matrix.row(r)) pending.emplace_back(r, c);
    std::sort(pending.begin(), pending.end());
    pending.erase(std::unique(pending.begin(), pending.end()), pending.end());
    std::vector<std::uint64_t> row_ptr(dim + 1, 0), col_idx;
    col_idx.reserve(pending.size());
    for (const auto& [r, c] : pending) {
        row_ptr[r + 1]++;
        col_idx.push_back(c);
    }
    for (std::uint64_t r = 0; r < dim; ++r) row_ptr[r + 1] += row_ptr[r];
    pending.clear();
    pending.shrink_to_fit();
    slot.matrix = SparseMatrix::from_parts(dim, dim, std::move(row_ptr), std::move(col_idx));
    slot.device.clear();
    slot.transposed.reset();
}

void PropertyGraph::flush() const {
    for (auto& [name, slot] : relations_) {
        (void)name;
        flush_slot(slot, capacity_);
    }
    flush_slot(any_, capacity_);
}

const PropertyGraph::Slot* PropertyGraph::find_slot(const RelationRef& rel) const {
    if (rel.is_any()) return &any_;
    auto it = relations_.find(*rel.name);
    return it == relations_.end() ? nullptr : &it->second;
}

const SparseMatrix& PropertyGraph::relation_matrix(const RelationRef& rel) const {
    flush();
    const Slot* slot = find_slot(rel);
    return slot ? slot->matrix : empty_.matrix;
}

const SparseMatrix& PropertyGraph::transposed_matrix(const RelationRef& rel) const {
    flush();  // graph.cpp:90-102: lazily, under a mutex, cached until the next write
    const Slot* found = find_slot(rel);
    Slot& slot = const_cast<Slot&>(found ? *found : empty_);
    std::lock_guard lock(*device_mutex_);
    if (!slot.transposed) {
        const SparseMatrix& m = slot.matrix;  // counting sort by column (sparse.cpp:379-403)
        std::vector<std::uint64_t> rp(m.ncols() + 1, 0), ci(m.nvals());
        for (std::uint64_t c : m.col_idx()) rp[c + 1]++;
        for (std::uint64_t c = 0; c < m.ncols(); ++c) rp[c + 1] += rp[c];
        std::vector<std::uint64_t> pos(rp.begin(), rp.end() - 1);
        for (std::uint64_t r = 0; r < m.nrows(); ++r)
            for (std::uint64_t c : m.row(r)) ci[pos[c]++] = r;  // rows visited ascending
        slot.transposed = SparseMatrix::from_parts(m.ncols(), m.nrows(), std::move(rp), std::move(ci));
    }
    return *slot.transposed;
}

const DeviceMatrix& PropertyGraph::device_matrix(const RelationRef& rel, int device) const {
    flush();
    const Slot* found = find_slot(rel);
    Slot& slot = const_cast<Slot&>(found ? *found : empty_);
    std::lock_guard lock(*device_mutex_);
    auto it = slot.device.find(device);
    if (it != slot.device.end()) return *it->second;
    const SparseMatrix& m = slot.matrix;
    mgk_graph* h = nullptr;
    static const std::uint64_t kZero = 0;
    const int rc = mgk_graph_upload(device, m.nrows(), m.nvals(), m.row_ptr().data(),
                                    m.nvals() ? m.col_idx().data() : &kZero, &h);
    if (rc != MGK_OK) throw_mgk(rc);
    auto dm = std::make_shared<DeviceMatrix>(h);
    slot.device.emplace(device, dm);
    return *dm;
}

std::vector<std::string> PropertyGraph::relation_names() const {
    std::vector<std::string> names;
    for (const auto& [name, slot] : relations_) {
        (void)slot;
        names.push_back(name);
    }
    return names;
}

// ---- k-hop ------------------------------------------------------------------------------
namespace {
void check_query(const PropertyGraph& graph, std::uint64_t seed, std::uint32_t k) {
    if (seed >= graph.node_count())  // execute.cpp:348-354
        throw ContractError(fmt("k-hop seed %llu is not an allocated node", (unsigned long long)seed));
    if (k < 1 || k > kMaxHops)
        throw ContractError(fmt("k-hop count %u outside [1, %u]", k, kMaxHops));
}
}  // namespace

BitVector k_hop_frontier(const PropertyGraph& graph, const KHopQuery& query) {
    check_query(graph, query.seed, query.k);
    const DeviceMatrix& dm = graph.device_matrix(query.relation);
    const std::uint64_t dim = graph.capacity();
    std::vector<std::uint64_t> ids(dim);
    std::uint64_t n = 0;
    const int rc = mgk_khop_frontier(dm.handle(), query.seed, query.k,
                                     query.mode == TraverseMode::Exact ? MGK_EXACT : MGK_CUMULATIVE,
                                     ids.data(), ids.size(), &n);
    if (rc != MGK_OK) throw_mgk(rc);
    ids.resize(n);
    return BitVector::from_sorted(dim, std::move(ids));
}

std::uint64_t k_hop_count(const PropertyGraph& graph, const KHopQuery& query) {
    check_query(graph, query.seed, query.k);
    const std::uint64_t seed = query.seed;
    return k_hop_count_batch(graph, std::span<const std::uint64_t>(&seed, 1), query.k, query.relation,
                             query.mode)[0];
}

std::vector<std::uint64_t> k_hop_count_batch(const PropertyGraph& graph,
                                             std::span<const std::uint64_t> seeds, std::uint32_t k,
                                             const RelationRef& relation, TraverseMode mode) {
    for (std::uint64_t s : seeds) check_query(graph, s, k);
    if (seeds.empty()) {
        if (k < 1 || k > kMaxHops) throw ContractError(fmt("k-hop count %u outside [1, %u]", k, kMaxHops));
        return {};
    }
    const DeviceMatrix& dm = graph.device_matrix(relation);
    std::vector<std::uint64_t> counts(seeds.size());
    const int rc = mgk_khop_count(dm.handle(), seeds.data(), seeds.size(), k,
                                  mode == TraverseMode::Exact ? MGK_EXACT : MGK_CUMULATIVE, counts.data());
    if (rc != MGK_OK) throw_mgk(rc);
    return counts;
}

std::vector<std::uint64_t> walk_targets(const PropertyGraph& graph, std::uint64_t src, std::uint32_t min,
                                        std::uint32_t max, const RelationRef& relation) {
    const DeviceMatrix& dm = graph.device_matrix(relation);
    std::vector<std::uint64_t> ids(graph.capacity());
    std::uint64_t n = 0;
    const int rc = mgk_walk_targets(dm.handle(), src, min, max, ids.data(), ids.size(), &n);
    if (rc != MGK_OK) throw_mgk(rc);
    ids.resize(n);
    return ids;
}

std::vector<std::uint64_t> walk_count_batch(const PropertyGraph& graph, std::span<const std::uint64_t> sources,
                                            std::uint32_t min, std::uint32_t max, const RelationRef& relation) {
    const DeviceMatrix& dm = graph.device_matrix(relation);
    std::vector<std::uint64_t> counts(sources.size());
    const int rc = mgk_walk_count(dm.handle(), sources.data(), sources.size(), min, max, MGK_ENGINE_AUTO,
                                  counts.data());
    if (rc != MGK_OK) throw_mgk(rc);
    return counts;
}

// ---- harness -----------------------------------------------------------------------------
void RmatParams::validate() const {  // bench.cpp:96-105
    if (scale > 24) throw ContractError(fmt("RMAT scale %u exceeds the cap of 24", scale));
    if (a < 0 || b < 0 || c < 0 || d < 0)
        throw ContractError("RMAT quadrant probabilities must be non-negative");
    const double sum = a + b + c + d;
    if (std::abs(sum - 1.0) > 1e-9)
        throw ContractError("RMAT quadrant probabilities sum to " + format_double(sum) + ", expected 1");
}

EdgeList rmat_generate(const RmatParams& params) {  // bench.cpp:107-137 (same stream)
    params.validate();
    std::mt19937_64 rng(params.rng_seed);
    const double ab = params.a + params.b, abc = ab + params.c;
    EdgeList edges;
    edges.reserve(params.edge_count());
    for (std::uint64_t e = 0; e < params.edge_count(); ++e) {
        std::uint32_t src = 0, dst = 0;
        for (std::uint32_t level = 0; level < params.scale; ++level) {
            const double r = unit_double(rng);
            std::uint32_t sb = 0, db = 0;
            if (r < params.a) {
            } else if (r < ab) {
                db = 1;
            } else if (r < abc) {
                sb = 1;
            } else {
                sb = 1;
                db = 1;
            }
            src = (src << 1) | sb;
            dst = (dst << 1) | db;
        }
        edges.push_back({src, dst});
    }
    return edges;
}

EdgeList load_edge_list(const std::filesystem::path& path) {  // bench.cpp:139-173
    std::ifstream in(path, std::ios::binary);
    if (!in) throw HarnessError("cannot open edge list '" + path.string() + "'");
    constexpr std::uint32_t kIdCap = 1u << 24;
    EdgeList edges;
    std::string line;
    std::size_t line_no = 0;
    while (std::getline(in, line)) {
        ++line_no;
        if (!line.empty() && line.back() == '\r') line.pop_back();
        if (line.empty()) continue;
        const std::size_t tab = line.find('\t');
        if (tab == std::string::npos) throw HarnessError(fmt("edge list line %zu: expected 'src<TAB>dst'", line_no));
        std::uint32_t ids[2] = {0, 0};
        const char* bounds[3] = {line.data(), line.data() + tab + 1, line.data() + line.size()};
        for (int i = 0; i < 2; ++i) {
            const char* first = bounds[i];
            const char* last = i == 0 ? line.data() + tab : bounds[2];
            const auto [end, ec] = std::from_chars(first, last, ids[i]);
            if (ec != std::errc{} || end != last)
                throw HarnessError(fmt("edge list line %zu: malformed node id", line_no));
            if (ids[i] >= kIdCap)
                throw HarnessError(fmt("edge list line %zu: node id %u is at or above 2^24", line_no, ids[i]));
        }
        edges.push_back({ids[0], ids[1]});
    }
    if (in.bad()) throw HarnessError("I/O error reading '" + path.string() + "'");
    return edges;
}

std::uint64_t edge_list_node_count(const EdgeList& edges) {  // bench.cpp:175-183
    std::uint64_t max_id = 0;
    for (const auto& e : edges) max_id = std::max<std::uint64_t>(max_id, std::max(e.src, e.dst));
    return edges.empty() ? 0 : max_id + 1;
}

PropertyGraph build_bench_graph(const EdgeList& edges, std::uint64_t node_count) {  // bench.cpp:185-198
    PropertyGraph graph(std::max<std::uint64_t>(node_count, 1));
    for (std::uint64_t id = 0; id < node_count; ++id)
        graph.create_node({}, {{"id", Value(static_cast<std::int64_t>(id))}});
    const std::string relation(kBenchRelation);
    for (const auto& e : edges) {
        if (e.src >= node_count || e.dst >= node_count)
            throw ContractError(fmt("edge (%u, %u) outside the %llu-node range", e.src, e.dst,
                                    (unsigned long long)node_count));
        graph.create_edge(e.src, relation, e.dst);
    }
    graph.flush();
    return graph;
}

std::vector<std::uint64_t> pick_seeds(const PropertyGraph& graph, std::size_t n,
                                      std::uint64_t rng_seed) {  // bench.cpp:200-218
    const SparseMatrix& adjacency = graph.relation_matrix();
    std::vector<std::uint64_t> eligible;
    for (std::uint64_t id = 0; id < graph.node_count(); ++id)
        if (!adjacency.row(id).empty()) eligible.push_back(id);
    if (eligible.size() < n)
        throw HarnessError(fmt("need %zu seeds but only %zu nodes have out-degree >= 1", n,
                               eligible.size()));
    std::mt19937_64 rng(rng_seed);
    for (std::size_t i = 0; i < n; ++i) {
        const std::size_t j = i + static_cast<std::size_t>(bounded_draw(rng, eligible.size() - i));
        std::swap(eligible[i], eligible[j]);
    }
    eligible.resize(n);
    return eligible;
}

SectionStats summarize(const std::vector<SeedRun>& runs) {  // bench.cpp:271-295
    if (runs.empty()) throw ContractError("cannot summarize an empty run list");
    const std::size_t n = runs.size();
    std::vector<std::int64_t> elapsed;
    std::int64_t total_us = 0;
    std::uint64_t total_count = 0;
    for (const auto& run : runs) {
        elapsed.push_back(run.elapsed_us);
        total_us += run.elapsed_us;
        total_count += run.count;
    }
    std::sort(elapsed.begin(), elapsed.end());
    SectionStats s;
    s.mean_us = static_cast<double>(total_us) / static_cast<double>(n);
    s.median_us = n % 2 == 1 ? static_cast<double>(elapsed[n / 2])
                             : (static_cast<double>(elapsed[n / 2 - 1]) + static_cast<double>(elapsed[n / 2])) / 2.0;
    const std::size_t rank = (99 * n + 99) / 100;
    s.p99_us = static_cast<double>(elapsed[rank - 1]);
    s.mean_count = static_cast<double>(total_count) / static_cast<double>(n);
    return s;
}

void BenchSchedule::validate() const {  // bench.cpp:297-309
    if (ks.size() != seeds_per_k.size())
        throw ContractError(fmt("schedule pairs %zu hop counts with %zu seed counts", ks.size(),
                                seeds_per_k.size()));
    for (const std::uint32_t k : ks)
        if (k < 1 || k > kMaxHops) throw ContractError(fmt("hop count %u outside [1, %u]", k, kMaxHops));
    for (std::size_t i = 0; i < seeds_per_k.size(); ++i)
        if (seeds_per_k[i] == 0) throw ContractError(fmt("seed count for k=%u must be at least 1", ks[i]));
}

KHopReport run_khop_benchmark(const PropertyGraph& graph, const BenchSchedule& schedule) {
    return run_khop_benchmark(graph, schedule, false);
}

KHopReport run_khop_benchmark(const PropertyGraph& graph, const BenchSchedule& schedule, bool batched) {
    schedule.validate();
    KHopReport report{schedule.mode, {}};
    if (schedule.ks.empty()) return report;
    graph.flush();
    const std::size_t max_seeds = *std::max_element(schedule.seeds_per_k.begin(), schedule.seeds_per_k.end());
    const auto master = pick_seeds(graph, max_seeds, schedule.rng_seed);
    graph.device_matrix();  // upload outside the timed region
    for (std::size_t i = 0; i < schedule.ks.size(); ++i) {
        KHopSection section{schedule.ks[i], {}, {}};
        const std::size_t ns = schedule.seeds_per_k[i];
        if (batched) {
            const auto t0 = std::chrono::steady_clock::now();
            std::vector<std::uint64_t> counts;
            try {
                counts = k_hop_count_batch(graph, std::span(master.data(), ns), section.k,
                                           RelationRef::any(), schedule.mode);
            } catch (const Error& e) {
                throw HarnessError(fmt("k=%u seed=%llu: %s", section.k, (unsigned long long)master[0], e.what()));
            }
            const auto us = std::chrono::duration_cast<std::chrono::microseconds>(
                                std::chrono::steady_clock::now() - t0).count() / (std::int64_t)ns;
            for (std::size_t j = 0; j < ns; ++j) section.runs.push_back({master[j], counts[j], us});
        } else {
            for (std::size_t j = 0; j < ns; ++j) {
                const KHopQuery q{master[j], section.k, RelationRef::any(), schedule.mode};
                const auto t0 = std::chrono::steady_clock::now();
                std::uint64_t count = 0;
                try {
                    count = k_hop_count(graph, q);
                } catch (const Error& e) {
                    throw HarnessError(fmt("k=%u seed=%llu: %s", section.k, (unsigned long long)master[j], e.what()));
                }
                const auto t1 = std::chrono::steady_clock::now();
                section.runs.push_back(
                    {master[j], count, std::chrono::duration_cast<std::chrono::microseconds>(t1 - t0).count()});
            }
        }
        section.stats = summarize(section.runs);
        report.sections.push_back(std::move(section));
    }
    return report;
}

std::string report_csv_string(const KHopReport& report) {  // bench.cpp:387-401
    std::string out = "k,seed,count,elapsed_us\n";
    for (const auto& s : report.sections)
        for (const auto& r : s.runs)
            out += fmt("%u,%llu,%llu,%lld\n", s.k, (unsigned long long)r.seed, (unsigned long long)r.count,
                       (long long)r.elapsed_us);
    out += "k,n_seeds,mean_us,median_us,p99_us,mean_count\n";
    for (const auto& s : report.sections)
        out += fmt("%u,%zu,", s.k, s.runs.size()) + format_double(s.stats.mean_us) + "," +
               format_double(s.stats.median_us) + "," + format_double(s.stats.p99_us) + "," +
               format_double(s.stats.mean_count) + "\n";
    return out;
}

void report_csv(const KHopReport& report, const std::filesystem::path& path) {
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) throw HarnessError("cannot open '" + path.string() + "' for writing");
    const std::string text = report_csv_string(report);
    out.write(text.data(), static_cast<std::streamsize>(text.size()));
    out.flush();
    if (!out) throw HarnessError("failed writing '" + path.string() + "'");
}

}  // namespace matgraph

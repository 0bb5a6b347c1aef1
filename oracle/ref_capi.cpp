// TEST INFRASTRUCTURE ONLY — never linked into the product path.
//
// A plain C wrapper around the *unmodified* reference library (matgraph,
// compiled from /root/reference/proj/core/src with -Dmatgraph=matgraph_ref by
// oracle/Makefile into oracle/_ref/libmatgraph_ref.so). It exists so Python
// tests, golden-fixture generation and bench.py's reference arm can drive the
// reference's own code path through ctypes:
//   build_bench_graph      proj/core/src/bench.cpp:185-198
//   k_hop_count/frontier   proj/core/src/execute.cpp:347-375
//   pick_seeds             proj/core/src/bench.cpp:200-218
//   rmat_generate          proj/core/src/bench.cpp:107-137
//   BfsOracle::count       proj/core/src/bench.cpp:233-259
//   snapshot_from_string / snapshot_to_string   proj/core/src/snapshot.cpp:127-231
//   mxm                    proj/core/src/sparse.cpp:292-363
// Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
// --impl reference) may load this library.
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "matgraph/ast.hpp"
#include "matgraph/bench.hpp"
#include "matgraph/cypher.hpp"
#include "matgraph/plan.hpp"
#include "matgraph/error.hpp"
#include "matgraph/execute.hpp"
#include "matgraph/graph.hpp"
#include "matgraph/snapshot.hpp"
#include "matgraph/sparse.hpp"

using matgraph_ref::PropertyGraph;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
    g_err = e.what();
    if (dynamic_cast<const matgraph_ref::ContractError*>(&e)) return 1;
    if (dynamic_cast<const matgraph_ref::HarnessError*>(&e)) return 2;
    if (dynamic_cast<const matgraph_ref::Error*>(&e)) return 3;
    return 4;
}

matgraph_ref::TraverseMode to_mode(int mode) {
    return mode == 1 ? matgraph_ref::TraverseMode::Cumulative : matgraph_ref::TraverseMode::Exact;
}

matgraph_ref::RelationRef to_rel(const char* relation) {
    if (relation == nullptr) return matgraph_ref::RelationRef::any();
    return matgraph_ref::RelationRef(relation);
}

matgraph_ref::EdgeList to_edges(const uint32_t* src, const uint32_t* dst, uint64_t m) {
    matgraph_ref::EdgeList edges(m);
    for (uint64_t i = 0; i < m; ++i) edges[i] = {src[i], dst[i]};
    return edges;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// ---- graph construction -----------------------------------------------------

void* ref_graph_new(uint64_t capacity) { return new PropertyGraph(capacity); }

int ref_graph_create_nodes(void* g, uint64_t count) {
    try {
        auto* graph = static_cast<PropertyGraph*>(g);
        for (uint64_t i = 0; i < count; ++i) graph->create_node({});
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

int ref_graph_create_edge(void* g, uint64_t src, const char* relation, uint64_t dst) {
    try {
        static_cast<PropertyGraph*>(g)->create_edge(src, relation, dst);
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

int ref_build_bench_graph(const uint32_t* src, const uint32_t* dst, uint64_t m,
                          uint64_t node_count, void** out) {
    try {
        auto edges = to_edges(src, dst, m);
        *out = new PropertyGraph(matgraph_ref::build_bench_graph(edges, node_count));
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

// A node with labels ("a,b" or "") and a <props> field in snapshot encoding.
int ref_graph_create_node_full(void* g, const char* labels_csv, const char* props_field) {
    try {
        std::vector<std::string> labels;
        std::string csv(labels_csv);
        size_t start = 0;
        while (!csv.empty()) {
            const size_t pos = csv.find(',', start);
            labels.push_back(csv.substr(start, pos == std::string::npos ? std::string::npos : pos - start));
            if (pos == std::string::npos) break;
            start = pos + 1;
        }
        static_cast<PropertyGraph*>(g)->create_node(labels, matgraph_ref::decode_props(props_field));
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

int ref_graph_create_edge_props(void* g, uint64_t src, const char* relation, uint64_t dst,
                                const char* props_field) {
    try {
        static_cast<PropertyGraph*>(g)->create_edge(src, relation, dst, matgraph_ref::decode_props(props_field));
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

// snapshot_from_string over text[0, len) (text[len] must be readable: the
// reference may peek one byte past a props item, see make_golden.py).
int ref_snapshot_parse(const char* text, uint64_t len, void** out) {
    try {
        *out = new PropertyGraph(matgraph_ref::snapshot_from_string(std::string_view(text, len)));
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

// snapshot_to_string: size first (out may be NULL), then the bytes.
int ref_snapshot_to_string(void* g, char* out, uint64_t cap, uint64_t* n) {
    try {
        const std::string s = matgraph_ref::snapshot_to_string(*static_cast<PropertyGraph*>(g));
        *n = s.size();
        if (out && cap >= s.size()) std::memcpy(out, s.data(), s.size());
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

// mxm over from_parts operands (vals NULL = structural). Two calls: out
// arrays NULL -> *nnz and *valued; then the CSR (+ values when valued).
int ref_mxm(uint64_t a_nrows, uint64_t a_ncols, const uint64_t* a_rp, const uint64_t* a_ci, const int64_t* a_vals,
            uint64_t b_nrows, uint64_t b_ncols, const uint64_t* b_rp, const uint64_t* b_ci, const int64_t* b_vals,
            int semiring, uint64_t m_nrows, uint64_t m_ncols, const uint64_t* m_rp, const uint64_t* m_ci,
            uint64_t* nnz, int* valued, uint64_t* out_rp, uint64_t* out_ci, int64_t* out_vals) {
    try {
        using matgraph_ref::SparseMatrix;
        auto make = [](uint64_t nr, uint64_t nc, const uint64_t* rp, const uint64_t* ci, const int64_t* v) {
            std::vector<uint64_t> r(rp, rp + nr + 1), c(ci, ci + rp[nr]);
            std::vector<int64_t> vv;
            if (v) vv.assign(v, v + rp[nr]);
            return SparseMatrix::from_parts(nr, nc, std::move(r), std::move(c), std::move(vv));
        };
        const SparseMatrix a = make(a_nrows, a_ncols, a_rp, a_ci, a_vals);
        const SparseMatrix b = make(b_nrows, b_ncols, b_rp, b_ci, b_vals);
        const matgraph_ref::Semiring& sr = semiring == 0 ? matgraph_ref::Semiring::bool_or_and()
                                         : semiring == 1 ? matgraph_ref::Semiring::plus_times()
                                                         : matgraph_ref::Semiring::min_plus();
        SparseMatrix mask;
        if (m_rp) mask = make(m_nrows, m_ncols, m_rp, m_ci, nullptr);
        const SparseMatrix c = matgraph_ref::mxm(a, b, sr, m_rp ? &mask : nullptr);
        *nnz = c.nvals();
        *valued = c.valued() ? 1 : 0;
        if (out_rp) std::memcpy(out_rp, c.row_ptr().data(), (c.nrows() + 1) * 8);
        if (out_ci && c.nvals()) std::memcpy(out_ci, c.col_idx().data(), c.nvals() * 8);
        if (out_vals && c.valued() && c.nvals())
            for (uint64_t r = 0, p = 0; r < c.nrows(); ++r)
                for (int64_t v : c.row_values(r)) out_vals[p++] = v;
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

void ref_graph_free(void* g) { delete static_cast<PropertyGraph*>(g); }

uint64_t ref_graph_node_count(void* g) { return static_cast<PropertyGraph*>(g)->node_count(); }

// CSR of relation_matrix(rel): nrows + nnz first (row_ptr/col_idx may be NULL).
int ref_graph_relation_csr(void* g, const char* relation, uint64_t* nrows, uint64_t* nnz,
                           uint64_t* row_ptr, uint64_t* col_idx) {
    try {
        const auto& m = static_cast<PropertyGraph*>(g)->relation_matrix(to_rel(relation));
        *nrows = m.nrows();
        *nnz = m.nvals();
        if (row_ptr) std::memcpy(row_ptr, m.row_ptr().data(), (m.nrows() + 1) * 8);
        if (col_idx) std::memcpy(col_idx, m.col_idx().data(), m.nvals() * 8);
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

// ---- the hot path -------------------------------------------------------------

int ref_k_hop_count(void* g, uint64_t seed, uint32_t k, int mode, const char* relation,
                    uint64_t* out) {
    try {
        *out = matgraph_ref::k_hop_count(*static_cast<PropertyGraph*>(g),
                                         {seed, k, to_rel(relation), to_mode(mode)});
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

int ref_k_hop_frontier(void* g, uint64_t seed, uint32_t k, int mode, const char* relation,
                       uint64_t* ids, uint64_t cap, uint64_t* n) {
    try {
        auto v = matgraph_ref::k_hop_frontier(*static_cast<PropertyGraph*>(g),
                                              {seed, k, to_rel(relation), to_mode(mode)});
        *n = v.nvals();
        const auto idx = v.indices();
        for (uint64_t i = 0; i < idx.size() && i < cap; ++i) ids[i] = idx[i];
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

// Seed-parallel timing harness over the reference's k_hop_count (the
// reference's own server runs one whole query per worker thread,
// proj/core/src/server.cpp:417-432). Seeds are dealt round-robin from an
// atomic cursor; counts land in seed order; *elapsed_s is wall time.
int ref_k_hop_count_many(void* g, const uint64_t* seeds, uint64_t nseeds, uint32_t k, int mode,
                         int threads, uint64_t* counts, double* elapsed_s) {
    auto* graph = static_cast<PropertyGraph*>(g);
    try {
        graph->relation_matrix();  // flush once, outside the timed region
    } catch (const std::exception& e) { return fail(e); }
    if (threads < 1) threads = 1;
    std::atomic<uint64_t> cursor{0};
    std::atomic<int> status{0};
    std::string first_err;
    std::atomic<bool> err_taken{false};
    auto worker = [&] {
        for (;;) {
            const uint64_t i = cursor.fetch_add(1);
            if (i >= nseeds) return;
            try {
                counts[i] = matgraph_ref::k_hop_count(
                    *graph, {seeds[i], k, matgraph_ref::RelationRef::any(), to_mode(mode)});
            } catch (const std::exception& e) {
                if (!err_taken.exchange(true)) {
                    first_err = e.what();
                    status = 1;
                }
                return;
            }
        }
    };
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int t = 1; t < threads; ++t) pool.emplace_back(worker);
    worker();
    for (auto& t : pool) t.join();
    *elapsed_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (status != 0) g_err = first_err;
    return status;
}

// ---- the reference's kernels on a bare matrix ("wrapper bypassed") ----------
// For graphs too big for build_bench_graph on the host (BASELINE cfg4, 1.47B
// edges: ~70 GB of pending buffers): the reference's own
// SparseMatrix::from_parts (sparse.cpp:101-114, which validates the CSR) and
// the k_hop_frontier loop body (execute.cpp:355-370) over it — vxm with the
// complemented visited mask and ewise_union, exactly as k_hop_frontier calls
// them; only the PropertyGraph wrapper (relation_matrix) is bypassed.
void* ref_matrix_from_csr_u32(uint64_t n, const uint32_t* row_ptr, const uint32_t* col_idx) {
    try {
        const uint64_t m = row_ptr[n];
        std::vector<uint64_t> rp(row_ptr, row_ptr + n + 1), ci(col_idx, col_idx + m);
        return new matgraph_ref::SparseMatrix(
            matgraph_ref::SparseMatrix::from_parts(n, n, std::move(rp), std::move(ci)));
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

void ref_matrix_free(void* m) { delete static_cast<matgraph_ref::SparseMatrix*>(m); }

}  // extern "C"

namespace {
// execute.cpp:347-371 with adj given (the seed / k checks of :348-354 kept)
uint64_t matrix_k_hop_count(const matgraph_ref::SparseMatrix& adj, uint64_t seed, uint32_t k, int mode) {
    using matgraph_ref::BitVector;
    if (seed >= adj.nrows())
        throw matgraph_ref::ContractError("k-hop seed " + std::to_string(seed) + " is not an allocated node");
    if (k < 1 || k > matgraph_ref::kMaxHops)
        throw matgraph_ref::ContractError("k-hop count " + std::to_string(k) + " outside [1, 32]");
    const uint64_t dim = adj.nrows();
    BitVector frontier = BitVector::from_sorted(dim, {seed});
    BitVector visited = frontier;
    for (uint32_t hop = 1; hop <= k; ++hop) {
        frontier = matgraph_ref::vxm(frontier, adj, &visited, /*complement_mask=*/true);
        if (frontier.empty()) break;
        visited = matgraph_ref::ewise_union(visited, frontier);
    }
    if (mode == 0) return frontier.nvals();
    return visited.nvals() - 1;  // visited minus the seed (execute.cpp:364-370)
}

// A pool over (seed, k) jobs: one whole query per thread at a time, jobs taken
// in the order given (callers put the deep ones first). Returns 0 or the
// first failure (g_err set).
template <typename F>
int run_jobs(uint64_t njobs, int threads, double* elapsed_s, F&& one) {
    if (threads < 1) threads = 1;
    std::atomic<uint64_t> cursor{0};
    std::atomic<int> status{0};
    std::string first_err;
    std::atomic<bool> err_taken{false};
    auto worker = [&] {
        for (;;) {
            const uint64_t i = cursor.fetch_add(1);
            if (i >= njobs) return;
            try {
                one(i);
            } catch (const std::exception& e) {
                if (!err_taken.exchange(true)) {
                    first_err = e.what();
                    status = 1;
                }
                return;
            }
        }
    };
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int t = 1; t < threads; ++t) pool.emplace_back(worker);
    worker();
    for (auto& t : pool) t.join();
    *elapsed_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (status != 0) g_err = first_err;
    return status;
}
}  // namespace

extern "C" {

// jobs i = (seeds[i], ks[i]) on the bare matrix; counts[i] = k_hop_count
int ref_matrix_khop_jobs(void* m, const uint64_t* seeds, const uint32_t* ks, uint64_t njobs, int mode,
                         int threads, uint64_t* counts, double* elapsed_s) {
    const auto& adj = *static_cast<matgraph_ref::SparseMatrix*>(m);
    return run_jobs(njobs, threads, elapsed_s,
                    [&](uint64_t i) { counts[i] = matrix_k_hop_count(adj, seeds[i], ks[i], mode); });
}

// the same job pool over the full store: matgraph_ref::k_hop_count itself
int ref_graph_khop_jobs(void* g, const uint64_t* seeds, const uint32_t* ks, uint64_t njobs, int mode,
                        int threads, uint64_t* counts, double* elapsed_s) {
    auto* graph = static_cast<PropertyGraph*>(g);
    try {
        graph->relation_matrix();  // flush once, outside the timed region
    } catch (const std::exception& e) { return fail(e); }
    return run_jobs(njobs, threads, elapsed_s, [&](uint64_t i) {
        counts[i] = matgraph_ref::k_hop_count(
            *graph, {seeds[i], ks[i], matgraph_ref::RelationRef::any(), to_mode(mode)});
    });
}

// (pick_seeds, bench.cpp:200-218, takes a PropertyGraph: for a bare matrix
// callers use the oracle's restatement orc_pick_seeds_u32, pinned to the
// reference's seeds by tests/test_bench_oracle.py.)

// Runs a Cypher query through the reference's parse -> plan -> execute
// (proj/core/src/cypher.cpp, plan.cpp, execute.cpp:342-345) and returns the
// table's wire text (to_string). Used to pin walk_targets (VarLenTraverse).
int ref_cypher(void* g, const char* text, char* out, uint64_t cap, uint64_t* n) {
    try {
        auto& graph = *static_cast<PropertyGraph*>(g);
        const std::string t = matgraph_ref::to_string(
            matgraph_ref::execute(matgraph_ref::plan(matgraph_ref::parse(text), graph), graph));
        *n = t.size();
        if (out && cap) {
            const uint64_t k = std::min<uint64_t>(cap - 1, t.size());
            std::memcpy(out, t.data(), k);
            out[k] = 0;
        }
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

// ---- harness pieces -------------------------------------------------------------

int ref_pick_seeds(void* g, uint64_t n, uint64_t rng_seed, uint64_t* out) {
    try {
        auto seeds = matgraph_ref::pick_seeds(*static_cast<PropertyGraph*>(g), n, rng_seed);
        for (uint64_t i = 0; i < seeds.size(); ++i) out[i] = seeds[i];
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

int ref_rmat_generate(uint32_t scale, uint32_t edge_factor, double a, double b, double c,
                      double d, uint64_t rng_seed, uint32_t* src, uint32_t* dst,
                      uint64_t* m) {
    try {
        matgraph_ref::RmatParams p;
        p.scale = scale;
        p.edge_factor = edge_factor;
        p.a = a;
        p.b = b;
        p.c = c;
        p.d = d;
        p.rng_seed = rng_seed;
        p.validate();
        if (src == nullptr) {
            *m = p.edge_count();
            return 0;
        }
        auto edges = matgraph_ref::rmat_generate(p);
        *m = edges.size();
        for (uint64_t i = 0; i < edges.size(); ++i) {
            src[i] = edges[i].src;
            dst[i] = edges[i].dst;
        }
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

void* ref_bfs_oracle_new(const uint32_t* src, const uint32_t* dst, uint64_t m, uint64_t n) {
    try {
        return new matgraph_ref::BfsOracle(to_edges(src, dst, m), n);
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

int ref_bfs_oracle_count(void* o, uint64_t seed, uint32_t k, int mode, uint64_t* out) {
    try {
        *out = static_cast<matgraph_ref::BfsOracle*>(o)->count(seed, k, to_mode(mode));
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

void ref_bfs_oracle_free(void* o) { delete static_cast<matgraph_ref::BfsOracle*>(o); }

}  // extern "C"

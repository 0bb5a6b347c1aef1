// The C++ drop-in (namespace matgraph, include/matgraph_b200/khop.hpp) run
// against the reference's own test cases for the k-hop path and against the
// CPU oracle (oracle/khop_oracle.c, linked as the checker).
//   proj/tests/test_execute.cpp:32-47, 104-139   k-hop known answers and errors
//   proj/tests/test_bench.cpp:33-349              harness pieces, oracle agreement
//   proj/tests/acceptance/acceptance_main.cpp:53-88  c1 (20 RMAT graphs x 50 seeds)
// `test_dropin --cpu` runs only the cases that need no GPU.
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <random>
#include <set>
#include <string>
#include <vector>

#include "matgraph_b200/khop.hpp"
#include "mini_test.hpp"

extern "C" {  // oracle/khop_oracle.c (checker only)
typedef struct orc_adj orc_adj;
orc_adj* orc_adj_new(uint64_t n, uint64_t m, const uint32_t* src, const uint32_t* dst);
void orc_adj_free(orc_adj* g);
uint64_t orc_bfs_count(const orc_adj* g, uint64_t seed, uint32_t k, int mode);
uint64_t orc_mxm(uint64_t a_nrows, const uint64_t* a_rp, const uint64_t* a_ci, const int64_t* a_vals,
                 uint64_t b_ncols, const uint64_t* b_rp, const uint64_t* b_ci, const int64_t* b_vals,
                 int semiring, const uint64_t* m_rp, const uint64_t* m_ci,
                 uint64_t* out_rp, uint64_t* out_ci, int64_t* out_vals);
}

using namespace matgraph;

namespace {

PropertyGraph path4() {  // 0 -> 1 -> 2 -> 3 over relation R
    PropertyGraph g;
    for (int i = 0; i < 4; ++i) g.create_node({});
    for (std::uint64_t i = 0; i < 3; ++i) g.create_edge(i, "R", i + 1);
    return g;
}

PropertyGraph triangle() {  // 0 -> 1 -> 2 -> 0 over relation R
    PropertyGraph g;
    for (int i = 0; i < 3; ++i) g.create_node({});
    g.create_edge(0, "R", 1);
    g.create_edge(1, "R", 2);
    g.create_edge(2, "R", 0);
    return g;
}

struct Oracle {  // BfsOracle semantics over the raw edge list
    orc_adj* h;
    Oracle(const EdgeList& e, std::uint64_t n) {
        std::vector<uint32_t> s, d;
        for (auto& t : e) {
            s.push_back(t.src);
            d.push_back(t.dst);
        }
        if (s.empty()) {
            s.push_back(0);
            d.push_back(0);
        }
        h = orc_adj_new(n, e.size(), s.data(), d.data());
    }
    ~Oracle() { orc_adj_free(h); }
    std::uint64_t count(std::uint64_t seed, std::uint32_t k, TraverseMode m) const {
        return orc_bfs_count(h, seed, k, m == TraverseMode::Exact ? 0 : 1);
    }
};

}  // namespace

// ---- proj/tests/test_execute.cpp ------------------------------------------------------------
GPU_TEST_CASE("k-hop counts match the masked-BFS definition") {  // test_execute.cpp:104-120
    PropertyGraph path = path4();
    PropertyGraph tri = triangle();
    CHECK(k_hop_count(path, {.seed = 0, .k = 2, .mode = TraverseMode::Exact}) == 1);
    const auto frontier = k_hop_frontier(path, {.seed = 0, .k = 2});
    CHECK(std::vector<std::uint64_t>(frontier.indices().begin(), frontier.indices().end()) ==
          std::vector<std::uint64_t>{2});
    CHECK(k_hop_count(path, {.seed = 3, .k = 1, .mode = TraverseMode::Exact}) == 0);
    CHECK(k_hop_count(path, {.seed = 0, .k = 6, .mode = TraverseMode::Cumulative}) == 3);
    CHECK(k_hop_count(tri, {.seed = 0, .k = 3, .mode = TraverseMode::Exact}) == 0);
    CHECK(k_hop_count(tri, {.seed = 0, .k = 3, .mode = TraverseMode::Cumulative}) == 2);
}

GPU_TEST_CASE("k-hop respects the relation filter") {  // test_execute.cpp:122-129
    PropertyGraph g = path4();
    g.create_edge(0, "S", 3);
    CHECK(k_hop_count(g, {.seed = 0, .k = 1, .relation = "R"}) == 1);
    CHECK(k_hop_count(g, {.seed = 0, .k = 1, .relation = RelationRef::any()}) == 2);
    CHECK(k_hop_count(g, {.seed = 0, .k = 1, .relation = "S"}) == 1);
    CHECK(k_hop_count(g, {.seed = 0, .k = 1, .relation = "NONE"}) == 0);
}

TEST_CASE("k-hop rejects out-of-range seeds and hop counts") {  // test_execute.cpp:131-139
    PropertyGraph g = path4();
    CHECK_THROWS_WITH_AS(k_hop_count(g, {.seed = 99, .k = 1}), "k-hop seed 99 is not an allocated node",
                         ContractError);
    CHECK_THROWS_WITH_AS(k_hop_count(g, {.seed = 0, .k = 0}), "k-hop count 0 outside [1, 32]", ContractError);
    CHECK_THROWS_WITH_AS(k_hop_count(g, {.seed = 0, .k = 33}), "k-hop count 33 outside [1, 32]",
                         ContractError);
}

GPU_TEST_CASE("a cached device matrix is dropped when new edges arrive") {
    PropertyGraph g = path4();
    CHECK(k_hop_count(g, {.seed = 0, .k = 1}) == 1);
    g.create_edge(0, "R", 2);  // pending until the next read flushes it
    CHECK(k_hop_count(g, {.seed = 0, .k = 1}) == 2);
    CHECK(k_hop_count(g, {.seed = 0, .k = 2, .mode = TraverseMode::Exact}) == 1);
}

GPU_TEST_CASE("anchored variable-length walks agree with the in-process k-hop counts") {
    // test_execute.cpp:141-173: MATCH (a {id: S})-[*k..k]->(b) WHERE b.id <> S and
    // [*1..k] equal k_hop_count exact / cumulative; walk_targets (execute.cpp:43-60)
    // starts with nothing visited, so S is dropped by the WHERE term.
    PropertyGraph graphs[] = {path4(), triangle()};
    for (PropertyGraph& g : graphs) {
        for (std::uint64_t seed = 0; seed < g.node_count(); ++seed) {
            for (std::uint32_t k = 1; k <= 4; ++k) {
                auto without_seed = [&](std::vector<std::uint64_t> ids) {
                    return std::count_if(ids.begin(), ids.end(), [&](std::uint64_t v) { return v != seed; });
                };
                CHECK(without_seed(walk_targets(g, seed, k, k, "R")) ==
                      (long)k_hop_count(g, {.seed = seed, .k = k, .relation = "R", .mode = TraverseMode::Exact}));
                CHECK(without_seed(walk_targets(g, seed, 1, k, "R")) ==
                      (long)k_hop_count(g, {.seed = seed, .k = k, .relation = "R", .mode = TraverseMode::Cumulative}));
            }
        }
    }
    PropertyGraph tri = triangle();  // 0 -> 1 -> 2 -> 0: the source returns at hop 3
    CHECK(walk_targets(tri, 0, 3, 3, "R") == std::vector<std::uint64_t>{0});
    const std::uint64_t srcs[] = {0, 1, 2};
    CHECK(walk_count_batch(tri, srcs, 1, 3, "R") == std::vector<std::uint64_t>({3, 3, 3}));
    CHECK_THROWS_WITH_AS(walk_targets(tri, 0, 0, 2, "R"), "hop minimum must be at least 1", ContractError);
}

// ---- proj/tests/test_bench.cpp --------------------------------------------------------------
TEST_CASE("rmat generation is deterministic and in bounds") {  // test_bench.cpp:33-50
    RmatParams params;
    params.scale = 8;
    params.rng_seed = 42;
    const EdgeList first = rmat_generate(params);
    REQUIRE(first.size() == params.edge_count());
    CHECK(first == rmat_generate(params));
    params.rng_seed = 43;
    CHECK(rmat_generate(params) != first);
    for (const auto& e : first) REQUIRE(e.src < 256 && e.dst < 256);
}

TEST_CASE("rmat parameters are validated") {  // test_bench.cpp:66-79
    RmatParams params;
    params.scale = 25;
    CHECK_THROWS_WITH_AS(params.validate(), "RMAT scale 25 exceeds the cap of 24", ContractError);
    params.scale = 10;
    params.a = -0.1;
    params.b = 0.57 + 0.19 + 0.1 - 0.05;
    CHECK_THROWS_WITH_AS(params.validate(), "RMAT quadrant probabilities must be non-negative", ContractError);
}

TEST_CASE("the bench graph carries one edge relation and collapses duplicates") {  // :81-91
    const EdgeList edges = {{0, 1}, {1, 2}, {1, 2}, {2, 0}};
    PropertyGraph g = build_bench_graph(edges, 4);
    CHECK(g.node_count() == 4);
    CHECK(g.relation_names() == std::vector<std::string>{std::string(kBenchRelation)});
    CHECK(g.relation_matrix("EDGE").nvals() == 3);
    CHECK_THROWS_WITH_AS(build_bench_graph({{5, 9}}, 4), "edge (5, 9) outside the 4-node range", ContractError);
}

TEST_CASE("seed picking is deterministic and sticks to source nodes") {  // :93-102
    RmatParams params;
    params.scale = 7;
    PropertyGraph g = build_bench_graph(rmat_generate(params), params.node_count());
    const auto seeds = pick_seeds(g, 50, 9);
    CHECK(seeds == pick_seeds(g, 50, 9));
    CHECK(seeds != pick_seeds(g, 50, 10));
    CHECK(std::set<std::uint64_t>(seeds.begin(), seeds.end()).size() == seeds.size());
    for (auto s : seeds) CHECK_FALSE(g.relation_matrix().row(s).empty());
}

TEST_CASE("seed picking fails loudly when too few nodes qualify") {  // :104-113
    PropertyGraph g = build_bench_graph({{0, 1}}, 3);
    CHECK(pick_seeds(g, 1, 1) == std::vector<std::uint64_t>{0});
    CHECK_THROWS_WITH_AS(pick_seeds(g, 2, 1), "need 2 seeds but only 1 nodes have out-degree >= 1",
                         HarnessError);
}

GPU_TEST_CASE("the oracle agrees with the k-hop counter on rmat graphs") {  // :115-138
    RmatParams params;
    params.scale = 6;
    params.rng_seed = 3;
    const EdgeList edges = rmat_generate(params);
    PropertyGraph g = build_bench_graph(edges, params.node_count());
    Oracle oracle(edges, params.node_count());
    for (std::uint64_t seed : pick_seeds(g, 20, 5))
        for (std::uint32_t k : {1u, 2u, 3u, 6u})
            for (TraverseMode mode : {TraverseMode::Exact, TraverseMode::Cumulative})
                CHECK(k_hop_count(g, {.seed = seed, .k = k, .relation = std::string(kBenchRelation),
                                      .mode = mode}) == oracle.count(seed, k, mode));
}

TEST_CASE("summary statistics match hand-computed values") {  // :148-168
    std::vector<SeedRun> runs = {{0, 2, 10}, {1, 4, 30}, {2, 6, 20}, {3, 8, 40}};
    const SectionStats s = summarize(runs);
    CHECK(s.mean_us == 25.0);
    CHECK(s.median_us == 25.0);
    CHECK(s.p99_us == 40.0);
    CHECK(s.mean_count == 5.0);
    CHECK(summarize({{0, 0, 1}, {1, 0, 100}, {2, 0, 2}}).median_us == 2.0);
    CHECK_THROWS_WITH_AS(summarize({}), "cannot summarize an empty run list", ContractError);
}

TEST_CASE("schedules validate their shape before any work starts") {  // :170-188
    BenchSchedule schedule;
    schedule.ks = {1, 2};
    schedule.seeds_per_k = {10};
    CHECK_THROWS_WITH_AS(schedule.validate(), "schedule pairs 2 hop counts with 1 seed counts", ContractError);
    schedule.seeds_per_k = {10, 0};
    CHECK_THROWS_WITH_AS(schedule.validate(), "seed count for k=2 must be at least 1", ContractError);
    schedule.ks = {0, 2};
    schedule.seeds_per_k = {10, 10};
    CHECK_THROWS_WITH_AS(schedule.validate(), "hop count 0 outside [1, 32]", ContractError);
}

TEST_CASE("reports serialize with fixed headers and one row per unit") {  // :190-209
    KHopReport empty;
    CHECK(report_csv_string(empty) == "k,seed,count,elapsed_us\nk,n_seeds,mean_us,median_us,p99_us,mean_count\n");
    KHopReport report;
    report.sections.push_back({2, {{5, 7, 10}, {6, 9, 20}}, summarize({{5, 7, 10}, {6, 9, 20}})});
    CHECK(report_csv_string(report) ==
          "k,seed,count,elapsed_us\n2,5,7,10\n2,6,9,20\n"
          "k,n_seeds,mean_us,median_us,p99_us,mean_count\n2,2,15,15,20,8\n");
}

GPU_TEST_CASE("benchmark counts agree with the oracle in both modes") {  // :295-317
    RmatParams params;
    params.scale = 6;
    params.rng_seed = 11;
    const EdgeList edges = rmat_generate(params);
    PropertyGraph g = build_bench_graph(edges, params.node_count());
    Oracle oracle(edges, params.node_count());
    for (TraverseMode mode : {TraverseMode::Exact, TraverseMode::Cumulative})
        for (bool batched : {false, true}) {
            BenchSchedule schedule;
            schedule.ks = {1, 2, 6};
            schedule.seeds_per_k = {10, 10, 10};
            schedule.mode = mode;
            const KHopReport report = run_khop_benchmark(g, schedule, batched);
            for (const auto& section : report.sections)
                for (const auto& run : section.runs)
                    CHECK(run.count == oracle.count(run.seed, section.k, mode));
        }
}

// ---- acceptance c1 --------------------------------------------------------------------------
GPU_TEST_CASE("c1: 8000 k-hop counts equal the BFS oracle") {  // acceptance_main.cpp:53-88
    std::uint64_t agreements = 0, mismatches = 0;
    for (std::uint64_t rng_seed = 1; rng_seed <= 20; ++rng_seed) {
        RmatParams params;
        params.scale = static_cast<std::uint32_t>(6 + (rng_seed - 1) % 7);
        params.rng_seed = rng_seed;
        const EdgeList edges = rmat_generate(params);
        PropertyGraph graph = build_bench_graph(edges, params.node_count());
        Oracle oracle(edges, params.node_count());
        const auto seeds = pick_seeds(graph, 50, rng_seed);
        for (std::uint32_t k : {1u, 2u, 3u, 6u})
            for (TraverseMode mode : {TraverseMode::Exact, TraverseMode::Cumulative}) {
                const auto got = k_hop_count_batch(graph, seeds, k, std::string(kBenchRelation), mode);
                for (std::size_t i = 0; i < seeds.size(); ++i)
                    (got[i] == oracle.count(seeds[i], k, mode) ? agreements : mismatches) += 1;
            }
    }
    CHECK(mismatches == 0);
    CHECK(agreements == 8000);
}

// ---- mxm (proj/tests/test_sparse.cpp:165-243 shapes) --------------------------------------
namespace {
SparseMatrix build(std::uint64_t nr, std::uint64_t nc, std::vector<MatrixTuple> t, bool valued) {
    std::sort(t.begin(), t.end(), [](const MatrixTuple& x, const MatrixTuple& y) {
        return x.row != y.row ? x.row < y.row : x.col < y.col;
    });
    std::vector<std::uint64_t> rp(nr + 1, 0), ci;
    std::vector<std::int64_t> v;
    for (auto& x : t) {
        ++rp[x.row + 1];
        ci.push_back(x.col);
        if (valued) v.push_back(x.value);
    }
    for (std::uint64_t i = 0; i < nr; ++i) rp[i + 1] += rp[i];
    return SparseMatrix::from_parts(nr, nc, std::move(rp), std::move(ci), std::move(v));
}

SparseMatrix oracle_mxm(const SparseMatrix& a, const SparseMatrix& b, int sr, const SparseMatrix* mask) {
    auto vals = [](const SparseMatrix& m) { return m.valued() ? m.values().data() : nullptr; };
    const std::uint64_t nnz = orc_mxm(a.nrows(), a.row_ptr().data(), a.col_idx().data(), vals(a), b.ncols(),
                                      b.row_ptr().data(), b.col_idx().data(), vals(b), sr,
                                      mask ? mask->row_ptr().data() : nullptr,
                                      mask ? mask->col_idx().data() : nullptr, nullptr, nullptr, nullptr);
    std::vector<std::uint64_t> rp(a.nrows() + 1), ci(nnz);
    std::vector<std::int64_t> v(nnz);
    orc_mxm(a.nrows(), a.row_ptr().data(), a.col_idx().data(), vals(a), b.ncols(), b.row_ptr().data(),
            b.col_idx().data(), vals(b), sr, mask ? mask->row_ptr().data() : nullptr,
            mask ? mask->col_idx().data() : nullptr, rp.data(), ci.data(), v.data());
    if (sr == 0 || nnz == 0) v.clear();
    return SparseMatrix::from_parts(a.nrows(), b.ncols(), std::move(rp), std::move(ci), std::move(v));
}
}  // namespace

GPU_TEST_CASE("mxm hand examples") {
    const SparseMatrix path = build(4, 4, {{0, 1}, {1, 2}, {2, 3}}, false);
    const SparseMatrix two = mxm(path, path);
    CHECK(nvals(two) == 2);
    CHECK(two.contains(0, 2));
    CHECK(two.contains(1, 3));
    CHECK(!two.valued());
    const SparseMatrix a = build(2, 2, {{0, 0, 1}, {0, 1, 2}, {1, 1, 3}}, true);
    const SparseMatrix b = build(2, 2, {{0, 0, 4}, {1, 0, 5}, {1, 1, 6}}, true);
    const auto t = mxm(a, b, Semiring::plus_times()).extract_tuples();
    REQUIRE(t.size() == 4);
    CHECK(t[0] == (MatrixTuple{0, 0, 14}));
    CHECK(t[1] == (MatrixTuple{0, 1, 12}));
    CHECK(t[2] == (MatrixTuple{1, 0, 15}));
    CHECK(t[3] == (MatrixTuple{1, 1, 18}));
    const SparseMatrix d = build(3, 3, {{0, 1, 5}, {1, 2, 2}, {0, 2, 9}}, true);
    const auto dist = mxm(d, d, Semiring::min_plus()).extract_tuples();
    REQUIRE(dist.size() == 1);
    CHECK(dist[0] == (MatrixTuple{0, 2, 7}));
    CHECK_THROWS_WITH_AS(mxm(a, build(3, 3, {}, false)), "mxm: inner dimensions disagree (2x2 times 3x3)",
                         ContractError);
    const SparseMatrix pattern = build(3, 3, {{0, 1}, {1, 2}}, false);
    const auto counted = mxm(pattern, pattern, Semiring::plus_times()).extract_tuples();
    REQUIRE(counted.size() == 1);
    CHECK(counted[0] == (MatrixTuple{0, 2, 1}));
}

GPU_TEST_CASE("mxm mask restricts the result pattern") {
    const SparseMatrix path = build(4, 4, {{0, 1}, {1, 2}, {2, 3}}, false);
    const SparseMatrix mask = build(4, 4, {{0, 2}}, false);
    const SparseMatrix two = mxm(path, path, Semiring::bool_or_and(), &mask);
    CHECK(nvals(two) == 1);
    CHECK(two.contains(0, 2));
    const SparseMatrix bad = build(3, 4, {}, false);
    CHECK_THROWS_WITH_AS(mxm(path, path, Semiring::bool_or_and(), &bad),
                         "mxm: mask shape 3x4 != result shape 4x4", ContractError);
}

GPU_TEST_CASE("mxm agrees with the C oracle across semirings") {
    std::mt19937_64 rng(202);
    const Semiring* rings[] = {&Semiring::bool_or_and(), &Semiring::plus_times(), &Semiring::min_plus()};
    for (int trial = 0; trial < 90; ++trial) {
        const std::uint64_t m = 1 + rng() % 20, k = 1 + rng() % 20, n = 1 + rng() % 20;
        const int sr = trial % 3;
        const double dens[] = {0.02, 0.1, 0.35};
        const double d = dens[(trial / 3) % 3];
        auto rand_t = [&](std::uint64_t nr, std::uint64_t nc, double p) {
            std::vector<MatrixTuple> t;
            for (std::uint64_t i = 0; i < nr; ++i)
                for (std::uint64_t j = 0; j < nc; ++j)
                    if ((double)(rng() >> 11) * 0x1.0p-53 < p) t.push_back({i, j, (std::int64_t)(rng() % 101) - 50});
            return t;
        };
        const SparseMatrix a = build(m, k, rand_t(m, k, d), sr != 0), b = build(k, n, rand_t(k, n, d), sr != 0);
        const SparseMatrix mask = build(m, n, rand_t(m, n, 0.5), false);
        const SparseMatrix* mp = trial % 4 == 0 ? &mask : nullptr;
        const SparseMatrix got = mxm(a, b, *rings[sr], mp), want = oracle_mxm(a, b, sr, mp);
        CHECK(got.extract_tuples() == want.extract_tuples());
        CHECK(got.valued() == want.valued());
    }
}

int main(int argc, char** argv) { return mini::run(argc, argv); }

// ---- the rest of the reference's graph-load / harness signatures ------------------------
TEST_CASE("create_node / create_edge accept labels and PropertyMap (graph.cpp:31-82)") {
    PropertyGraph g;
    for (std::int64_t i = 0; i < 4; ++i) g.create_node({}, {{"id", Value(i)}});
    const std::uint64_t tagged = g.create_node({"Person", "Admin"}, {{"name", Value("ann")}, {"age", Value(41)}});
    CHECK(tagged == 4);
    CHECK(g.node_props(2).at("id") == Value(std::int64_t{2}));
    CHECK(g.node_props(4).at("name").as_string() == "ann");
    CHECK((g.node_labels(4) == std::vector<std::string>{"Admin", "Person"}));
    g.create_edge(0, "R", 1, {{"w", Value(1.5)}});
    CHECK(g.edge_props(0, "R", 1) && g.edge_props(0, "R", 1)->at("w").as_float() == 1.5);
    g.create_edge(0, "R", 1);  // re-created without properties: the stored map is dropped
    CHECK(g.edge_props(0, "R", 1) == nullptr);
    CHECK_THROWS_WITH_AS(g.create_node({}, {{"bad key", Value(1)}}), "property key 'bad key' is not a valid identifier",
                         ContractError);
    CHECK_THROWS_WITH_AS(g.create_edge(0, "R", 1, {{"9x", Value(1)}}), "property key '9x' is not a valid identifier",
                         ContractError);
    CHECK(g.relation_matrix("R").nvals() == 1);
}

TEST_CASE("transposed_matrix is the CSR of A^T, cached until the next write (graph.cpp:90-102)") {
    PropertyGraph g = path4();
    g.create_edge(3, "R", 0);
    const SparseMatrix& t = g.transposed_matrix("R");
    CHECK(t.nrows() == g.relation_matrix("R").ncols());
    for (std::uint64_t r = 0; r < 4; ++r)
        for (std::uint64_t c = 0; c < 4; ++c) CHECK(t.contains(c, r) == g.relation_matrix("R").contains(r, c));
    CHECK(&g.transposed_matrix("R") == &t);  // cached
    g.create_edge(1, "R", 3);
    CHECK(g.transposed_matrix("R").contains(3, 1));  // invalidated by the write
    CHECK(g.transposed_matrix("NONE").nvals() == 0);
}

TEST_CASE("load_edge_list / edge_list_node_count (bench.cpp:139-183)") {
    const auto dir = std::filesystem::temp_directory_path();
    auto write = [&](const char* name, const std::string& text) {
        const auto p = dir / name;
        std::ofstream(p, std::ios::binary) << text;
        return p;
    };
    const auto ok = write("mgk_el_ok.tsv", "0\t1\r\n\n5\t2\n");
    const EdgeList e = load_edge_list(ok);
    CHECK((e == EdgeList{{0, 1}, {5, 2}}));
    CHECK(edge_list_node_count(e) == 6);
    CHECK(edge_list_node_count({}) == 0);
    CHECK_THROWS_WITH_AS(load_edge_list(write("mgk_el_a.tsv", "0\t1\n0 1\n")),
                         "edge list line 2: expected 'src<TAB>dst'", HarnessError);
    CHECK_THROWS_WITH_AS(load_edge_list(write("mgk_el_b.tsv", "0\tx\n")), "edge list line 1: malformed node id",
                         HarnessError);
    CHECK_THROWS_WITH_AS(load_edge_list(write("mgk_el_c.tsv", "16777216\t1\n")),
                         "edge list line 1: node id 16777216 is at or above 2^24", HarnessError);
    CHECK_THROWS_AS(load_edge_list(dir / "mgk_el_missing.tsv"), HarnessError);
}

TEST_CASE("BfsOracle (test infrastructure) keeps the reference's contract") {
    const EdgeList e{{0, 1}, {1, 2}, {2, 0}};
    BfsOracle o(e, 3);
    CHECK(o.node_count() == 3);
    CHECK(o.count(0, 1, TraverseMode::Exact) == 1);
    CHECK(o.count(0, 3, TraverseMode::Cumulative) == 2);
    CHECK_THROWS_WITH_AS(o.count(3, 1, TraverseMode::Exact), "oracle seed 3 is out of range", ContractError);
    CHECK_THROWS_WITH_AS(o.count(0, 33, TraverseMode::Exact), "oracle hop count 33 outside [1, 32]", ContractError);
    CHECK_THROWS_WITH_AS(BfsOracle(EdgeList{{0, 5}}, 3), "edge (0, 5) outside the 3-node range", ContractError);
}

GPU_TEST_CASE("run_khop_benchmark(graph, schedule): the reference's two-argument signature, checked by BfsOracle") {
    RmatParams p;
    p.scale = 9;
    p.rng_seed = 4;
    const EdgeList edges = rmat_generate(p);
    PropertyGraph g = build_bench_graph(edges, p.node_count());
    CHECK(g.node_props(7).at("id") == Value(std::int64_t{7}));  // bench.cpp:187-188
    BfsOracle oracle(edges, p.node_count());
    BenchSchedule s;
    s.ks = {1, 2, 3, 6};
    s.seeds_per_k = {20, 20, 5, 5};
    const KHopReport r = run_khop_benchmark(g, s);
    CHECK(r.sections.size() == 4);
    for (const auto& sec : r.sections)
        for (const auto& run : sec.runs) CHECK(run.count == oracle.count(run.seed, sec.k, TraverseMode::Exact));
    CHECK(bfs_oracle(g, r.sections[0].runs[0].seed, 2, TraverseMode::Cumulative) ==
          oracle.count(r.sections[0].runs[0].seed, 2, TraverseMode::Cumulative));
}

// The reference-side binding of the B200 engine (see mgk_bind.hpp and
// INTEGRATION.md §B). Compiled against the reference's own headers; routes
//   matgraph::k_hop_count / k_hop_frontier   (execute.cpp:347-375, via ld --wrap)
//   Executor::apply(VarLenTraverseOp)'s walk (execute.cpp:43-60, 110-116, via
//                                             mgk_bind::walk_targets)
// to libmgk.so (include/mgk.h). Matrices are uploaded once and cached by
// identity and contents; errors keep the reference's classes and messages.
#include "mgk_bind.hpp"

#include <atomic>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "matgraph/error.hpp"
#include "matgraph/execute.hpp"
#include "mgk.h"

using matgraph::BitVector;
using matgraph::KHopQuery;
using matgraph::PropertyGraph;
using matgraph::SparseMatrix;

namespace {

struct Routed {
    std::atomic<unsigned long long> count{0}, frontier{0}, walks{0}, uploads{0};
    ~Routed() {
        std::fprintf(stderr, "[mgk-bind] routed to the GPU: k_hop_count %llu, k_hop_frontier %llu, walks %llu "
                             "(device matrices uploaded: %llu)\n",
                     count.load(), frontier.load(), walks.load(), uploads.load());
    }
} routed;

[[noreturn]] void throw_mgk(int rc) {
    const std::string msg = mgk_last_error();
    if (rc == MGK_ECONTRACT || rc == MGK_ERANGE) throw matgraph::ContractError(msg);
    if (rc == MGK_EHARNESS) throw matgraph::HarnessError(msg);
    throw matgraph::Error(msg);
}

// One uploaded matrix. Identified by address AND contents (a matrix freed and
// re-created at the same address with other entries must not hit): a full
// host copy is kept for comparison.
struct Entry {
    const SparseMatrix* addr = nullptr;
    std::vector<std::uint64_t> rp, ci;
    mgk_graph* fwd = nullptr;
    mgk_graph* bwd = nullptr;  // transpose, built on the device on first use
    ~Entry() {
        if (fwd) mgk_graph_free(fwd);
        if (bwd) mgk_graph_free(bwd);
    }
};
std::mutex g_mu;
std::vector<std::unique_ptr<Entry>> g_cache;  // most recent last
constexpr std::size_t kCacheCap = 8;

bool same(const Entry& e, const SparseMatrix& a) {
    const auto rp = a.row_ptr();
    const auto ci = a.col_idx();
    return e.addr == &a && e.rp.size() == rp.size() && e.ci.size() == ci.size() &&
           std::memcmp(e.rp.data(), rp.data(), rp.size() * 8) == 0 &&
           (ci.empty() || std::memcmp(e.ci.data(), ci.data(), ci.size() * 8) == 0);
}

mgk_graph* device_of(const SparseMatrix& a, bool transposed) {
    std::lock_guard<std::mutex> lk(g_mu);
    Entry* hit = nullptr;
    for (auto it = g_cache.begin(); it != g_cache.end(); ++it)
        if (same(**it, a)) {
            std::rotate(it, it + 1, g_cache.end());
            hit = g_cache.back().get();
            break;
        }
    if (!hit) {
        auto e = std::make_unique<Entry>();
        e->addr = &a;
        e->rp.assign(a.row_ptr().begin(), a.row_ptr().end());
        e->ci.assign(a.col_idx().begin(), a.col_idx().end());
        static const std::uint64_t kZero = 0;
        const int rc = mgk_graph_upload(0, a.nrows(), a.nvals(), e->rp.data(), e->ci.empty() ? &kZero : e->ci.data(),
                                        &e->fwd);
        if (rc != MGK_OK) throw_mgk(rc);
        routed.uploads++;
        if (g_cache.size() == kCacheCap) g_cache.erase(g_cache.begin());
        g_cache.push_back(std::move(e));
        hit = g_cache.back().get();
    }
    if (!transposed) return hit->fwd;
    if (!hit->bwd) {
        const int rc = mgk_graph_transpose(hit->fwd, &hit->bwd);
        if (rc != MGK_OK) throw_mgk(rc);
    }
    return hit->bwd;
}

void check_query(const PropertyGraph& graph, const KHopQuery& q) {  // execute.cpp:348-354
    if (q.seed >= graph.node_count())
        throw matgraph::ContractError("k-hop seed " + std::to_string(q.seed) + " is not an allocated node");
    if (q.k < 1 || q.k > matgraph::kMaxHops)
        throw matgraph::ContractError("k-hop count " + std::to_string(q.k) + " outside [1, " +
                                      std::to_string(matgraph::kMaxHops) + "]");
}

int mode_of(const KHopQuery& q) { return q.mode == matgraph::TraverseMode::Exact ? MGK_EXACT : MGK_CUMULATIVE; }

}  // namespace

// ---- link-time replacements (GNU ld --wrap=<mangled name>) ------------------------------
std::uint64_t mgk_wrap_k_hop_count(const PropertyGraph& graph, const KHopQuery& q) __asm__(
    "__wrap__ZN8matgraph11k_hop_countERKNS_13PropertyGraphERKNS_9KHopQueryE");
BitVector mgk_wrap_k_hop_frontier(const PropertyGraph& graph, const KHopQuery& q) __asm__(
    "__wrap__ZN8matgraph14k_hop_frontierERKNS_13PropertyGraphERKNS_9KHopQueryE");

std::uint64_t mgk_wrap_k_hop_count(const PropertyGraph& graph, const KHopQuery& q) {
    check_query(graph, q);
    mgk_graph* h = device_of(graph.relation_matrix(q.relation), false);
    std::uint64_t out = 0;
    const int rc = mgk_khop_count(h, &q.seed, 1, q.k, mode_of(q), &out);
    if (rc != MGK_OK) throw_mgk(rc);
    routed.count++;
    return out;
}

BitVector mgk_wrap_k_hop_frontier(const PropertyGraph& graph, const KHopQuery& q) {
    check_query(graph, q);
    const SparseMatrix& adj = graph.relation_matrix(q.relation);
    mgk_graph* h = device_of(adj, false);
    std::vector<std::uint64_t> ids(adj.nrows());
    std::uint64_t n = 0;
    const int rc = mgk_khop_frontier(h, q.seed, q.k, mode_of(q), ids.data(), ids.size(), &n);
    if (rc != MGK_OK) throw_mgk(rc);
    ids.resize(n);
    routed.frontier++;
    return BitVector::from_sorted(adj.nrows(), std::move(ids));
}

// ---- the VarLenTraverseOp step -----------------------------------------------------------------
std::vector<std::uint64_t> mgk_bind::walk_targets(const PropertyGraph& graph, const matgraph::RelationRef& rel,
                                                  matgraph::Direction dir, const SparseMatrix& adj, std::uint64_t src,
                                                  std::uint32_t min, std::uint32_t max) {
    mgk_graph* h = device_of(graph.relation_matrix(rel), dir == matgraph::Direction::In);
    std::vector<std::uint64_t> ids(adj.nrows());
    std::uint64_t n = 0;
    const int rc = mgk_walk_targets(h, src, min, max, ids.data(), ids.size(), &n);
    if (rc != MGK_OK) throw_mgk(rc);
    ids.resize(n);
    routed.walks++;
    return ids;
}

// TEST INFRASTRUCTURE ONLY — matgraph::BfsOracle / bfs_oracle (bench.hpp:73-91,
// bench.cpp:220-269) for test binaries that link the C++ drop-in
// (libmatgraph_b200.so declares the class; only this file defines it). The BFS
// itself is the C oracle's queue BFS (khop_oracle.c orc_bfs_count), with the
// reference's contract checks and messages. Never linked into the product.
#include <cstdio>
#include <limits>
#include <string>

#include "matgraph_b200/khop.hpp"

extern "C" {
struct orc_adj;
orc_adj* orc_adj_new(std::uint64_t n, std::uint64_t m, const std::uint32_t* src, const std::uint32_t* dst);
void orc_adj_free(orc_adj* g);
std::uint64_t orc_bfs_count(const orc_adj* g, std::uint64_t seed, std::uint32_t k, int mode);
}

namespace matgraph {

BfsOracle::BfsOracle(const EdgeList& edges, std::uint64_t node_count) : node_count_(node_count) {
    if (node_count > std::numeric_limits<std::uint32_t>::max())
        throw ContractError("oracle supports at most 2^32 nodes, got " + std::to_string(node_count));
    std::vector<std::uint32_t> src, dst;
    src.reserve(edges.size());
    dst.reserve(edges.size());
    for (const auto& e : edges) {
        if (e.src >= node_count || e.dst >= node_count)
            throw ContractError("edge (" + std::to_string(e.src) + ", " + std::to_string(e.dst) + ") outside the " +
                                std::to_string(node_count) + "-node range");
        src.push_back(e.src);
        dst.push_back(e.dst);
    }
    impl_ = orc_adj_new(node_count, src.size(), src.data(), dst.data());
}

BfsOracle::~BfsOracle() {
    if (impl_) orc_adj_free(static_cast<orc_adj*>(impl_));
}

BfsOracle::BfsOracle(BfsOracle&& o) noexcept : impl_(o.impl_), node_count_(o.node_count_) { o.impl_ = nullptr; }

BfsOracle& BfsOracle::operator=(BfsOracle&& o) noexcept {
    if (this != &o) {
        if (impl_) orc_adj_free(static_cast<orc_adj*>(impl_));
        impl_ = o.impl_;
        node_count_ = o.node_count_;
        o.impl_ = nullptr;
    }
    return *this;
}

std::uint64_t BfsOracle::count(std::uint64_t seed, std::uint32_t k, TraverseMode mode) const {
    if (seed >= node_count_) throw ContractError("oracle seed " + std::to_string(seed) + " is out of range");
    if (k < 1 || k > kMaxHops)
        throw ContractError("oracle hop count " + std::to_string(k) + " outside [1, " + std::to_string(kMaxHops) + "]");
    return orc_bfs_count(static_cast<const orc_adj*>(impl_), seed, k, mode == TraverseMode::Exact ? 0 : 1);
}

std::uint64_t bfs_oracle(const PropertyGraph& graph, std::uint64_t seed, std::uint32_t k, TraverseMode mode) {
    graph.flush();
    EdgeList edges;
    for (const auto& t : graph.relation_matrix().extract_tuples())
        edges.push_back({static_cast<std::uint32_t>(t.row), static_cast<std::uint32_t>(t.col)});
    return BfsOracle(edges, graph.node_count()).count(seed, k, mode);
}

}  // namespace matgraph

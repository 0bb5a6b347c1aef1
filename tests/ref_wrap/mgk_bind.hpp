// The reference-side binding of the B200 engine: what a
// matgraph maintainer adds to route the k-hop hot path and the Cypher
// variable-length step to libmgk.so. Compiled against the REFERENCE's own
// headers (namespace matgraph); test infrastructure of this repo.
//
//  * k_hop_count / k_hop_frontier (execute.cpp:347-375): replaced at link
//    time with GNU ld --wrap (no reference source changes): the definitions
//    __wrap_<mangled name> live in mgk_bind.cpp.
//  * Executor::apply(VarLenTraverseOp) (execute.cpp:110-116) calls
//    mgk_bind::walk_targets instead of the file-local walk_targets
//    (execute.cpp:43-60): a one-line patch (INTEGRATION.md shows it), applied
//    by tests/ref_wrap/Makefile to a build-time copy of execute.cpp.
#pragma once

#include <cstdint>
#include <vector>

#include "matgraph/ast.hpp"
#include "matgraph/graph.hpp"
#include "matgraph/sparse.hpp"

namespace mgk_bind {

/// walk_targets(adj, src, min, max) on the GPU: the device copy of
/// relation_matrix(rel) walks forward (Direction::Out) or, for `<-`
/// patterns, its transpose built on the device (mgk_graph_transpose).
/// `adj` is the matrix the executor resolved (used for its dimension).
std::vector<std::uint64_t> walk_targets(const matgraph::PropertyGraph& graph, const matgraph::RelationRef& rel,
                                        matgraph::Direction dir, const matgraph::SparseMatrix& adj,
                                        std::uint64_t src, std::uint32_t min, std::uint32_t max);

}  // namespace mgk_bind

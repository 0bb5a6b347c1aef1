// Runs the reference's own Cypher stack (parse -> plan -> execute,
// cypher.cpp / plan.cpp / execute.cpp) on the graphs of
// tests/golden/walk_pins.json, with the variable-length step bound to the GPU
// (mgk_bind::walk_targets). Prints one JSON line per query:
//   {"graph": "s<scale>r<rng>" | "cycle_loop", "seed": S, "min": a, "max": b,
//    "dir": "out" | "in", "ids": [...]}
// tests/test_ref_wrap.py compares them with the reference-generated goldens.
#include <cstdio>
#include <string>
#include <vector>

#include "matgraph/bench.hpp"
#include "matgraph/cypher.hpp"
#include "matgraph/execute.hpp"
#include "matgraph/graph.hpp"
#include "matgraph/plan.hpp"

using namespace matgraph;

namespace {

std::string ids_json(const std::string& table) {  // "b\n#3\n#7\n" -> [3,7]
    std::string out = "[";
    std::size_t at = table.find('\n');
    bool first = true;
    while (at != std::string::npos && at + 1 < table.size()) {
        const std::size_t end = table.find('\n', at + 1);
        const std::string cell = table.substr(at + 1, end - at - 1);
        if (!cell.empty()) {
            out += (first ? "" : ",") + cell.substr(1);
            first = false;
        }
        at = end;
    }
    return out + "]";
}

void run(PropertyGraph& g, const std::string& name, std::uint64_t s, std::uint32_t lo, std::uint32_t hi) {
    for (const char* dir : {"out", "in"}) {
        const std::string pat = std::string(dir) == "out" ? "-[*" + std::to_string(lo) + ".." + std::to_string(hi) + "]->"
                                                          : "<-[*" + std::to_string(lo) + ".." + std::to_string(hi) + "]-";
        const std::string q = "MATCH (a {id: " + std::to_string(s) + "})" + pat + "(b) RETURN b";
        const std::string t = to_string(execute(plan(parse(q), g), g));
        std::printf("{\"graph\": \"%s\", \"seed\": %llu, \"min\": %u, \"max\": %u, \"dir\": \"%s\", \"ids\": %s}\n",
                    name.c_str(), (unsigned long long)s, lo, hi, dir, ids_json(t).c_str());
    }
}

}  // namespace

int main() {
    const std::uint32_t ranges[][2] = {{1, 1}, {1, 2}, {2, 2}, {1, 3}, {2, 4}, {3, 3}, {3, 6}, {1, 32}};
    const std::uint32_t graphs[][2] = {{6, 3}, {7, 8}, {8, 2}, {9, 17}};
    for (const auto& gs : graphs) {
        RmatParams p;
        p.scale = gs[0];
        p.rng_seed = gs[1];
        const EdgeList edges = rmat_generate(p);
        PropertyGraph g = build_bench_graph(edges, p.node_count());
        const std::string name = "s" + std::to_string(gs[0]) + "r" + std::to_string(gs[1]);
        for (std::uint64_t s : pick_seeds(g, 6, gs[1]))
            for (const auto& r : ranges) run(g, name, s, r[0], r[1]);
    }
    const EdgeList cyc{{0, 1}, {1, 2}, {2, 0}, {1, 1}, {2, 3}};
    PropertyGraph g = build_bench_graph(cyc, 4);
    const std::uint32_t cr[][2] = {{1, 1}, {1, 3}, {2, 2}, {3, 3}, {2, 5}};
    for (std::uint64_t s = 0; s < 4; ++s)
        for (const auto& r : cr) run(g, "cycle_loop", s, r[0], r[1]);
    return 0;
}

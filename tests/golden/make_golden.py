"""Regenerate the golden k-hop fixtures FROM THE REFERENCE ITSELF.

Run in the build container (needs /root/reference and oracle/_ref built):

    make -C oracle all && python tests/golden/make_golden.py

Every number written here comes out of the unmodified reference core
(oracle/_ref/libmatgraph_ref.so, compiled from /root/reference/proj/core/src)
through oracle/ref_capi.cpp:

* known_answers.json — the hand fixtures of proj/tests/test_execute.cpp:32-47
  (path4 0->1->2->3, triangle 0->1->2->0) with the k-hop counts, frontier and
  error strings the reference returns (pinned there at :104-139), plus the
  relation-filter case (:122-129).
* c1_sweep.json — the acceptance-c1 sweep (proj/tests/acceptance/
  acceptance_main.cpp:53-88): 20 RMAT graphs (scale 6 + (rng-1) % 7, rng 1..20),
  50 pick_seeds seeds each, k in {1,2,3,6}, exact + cumulative = 8000 counts,
  with a SHA-256 of each generated edge list and of its flushed CSR.
* harness_pins.json — rmat_generate / pick_seeds pins (proj/tests/
  test_bench.cpp:33-113 shapes) and a few sorted k_hop_frontier id lists.
* walk_pins.json — walk_targets (execute.cpp:43-60, the VarLenTraverse step)
  through the reference's own Cypher executor: counts and ids of
  MATCH (a {id: S})-[*min..max]->(b) on RMAT graphs and a cycle with a loop.

The GPU box never runs this script (no /root/reference there); it only reads
the committed JSON.
"""
from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import oracle  # noqa: E402

OUT = Path(__file__).resolve().parent
KS = (1, 2, 3, 6)


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def known_answers(R: oracle.Ref) -> dict:
    out = {}

    def path4():
        g = R.graph()
        g.create_nodes(4)
        for i in range(3):
            g.create_edge(i, "R", i + 1)
        return g

    def triangle():
        g = R.graph()
        g.create_nodes(3)
        g.create_edge(0, "R", 1)
        g.create_edge(1, "R", 2)
        g.create_edge(2, "R", 0)
        return g

    cases = []
    for name, make in (("path4", path4), ("triangle", triangle)):
        g = make()
        rp, ci = g.relation_csr()
        for seed in range(g.node_count):
            for k in (1, 2, 3, 4, 6, 32):
                for mode in (0, 1):
                    cases.append({
                        "graph": name, "seed": seed, "k": k, "mode": mode,
                        "count": g.k_hop_count(seed, k, mode),
                        "frontier": [int(x) for x in g.k_hop_frontier(seed, k, mode)],
                    })
        out[name] = {"node_count": g.node_count, "capacity": int(len(rp) - 1),
                     "row_ptr": [int(x) for x in rp], "col_idx": [int(x) for x in ci]}
    out["cases"] = cases

    # relation filter, test_execute.cpp:122-129 (path4 plus 0-[:S]->3)
    g = path4()
    g.create_edge(0, "S", 3)
    rel = {}
    for r in ("R", "S", "NONE", None):
        rp, ci = g.relation_csr(r)
        rel[str(r) if r else "ANY"] = {
            "row_ptr": [int(x) for x in rp], "col_idx": [int(x) for x in ci],
            "count_seed0_k1": g.k_hop_count(0, 1, 0, r),
        }
    out["relation_filter"] = rel

    # error strings, test_execute.cpp:131-139
    errs = []
    g = path4()
    for seed, k in ((99, 1), (0, 0), (0, 33), (4, 1)):
        try:
            g.k_hop_count(seed, k)
            errs.append({"seed": seed, "k": k, "error": None})
        except oracle.RefError as e:
            errs.append({"seed": seed, "k": k, "error": str(e), "kind": e.code})
    out["errors"] = errs
    return out


def c1_sweep(R: oracle.Ref) -> dict:
    graphs = []
    for rng_seed in range(1, 21):
        scale = 6 + (rng_seed - 1) % 7
        src, dst = R.rmat_generate(scale, rng_seed=rng_seed)
        n = 1 << scale
        g = R.build_bench_graph(src, dst, n)
        rp, ci = g.relation_csr()
        seeds = g.pick_seeds(50, rng_seed)
        counts = {}
        for mode in (0, 1):
            for k in KS:
                counts[f"{mode}_{k}"] = [g.k_hop_count(int(s), k, mode, "EDGE") for s in seeds]
        graphs.append({
            "rng_seed": rng_seed, "scale": scale, "node_count": n, "raw_edges": int(len(src)),
            "edges_sha256": sha(src, dst), "nnz": int(len(ci)), "csr_sha256": sha(rp, ci),
            "seeds": [int(s) for s in seeds], "counts": counts,
        })
    return {"ks": list(KS), "modes": ["exact", "cumulative"], "graphs": graphs}


def harness_pins(R: oracle.Ref) -> dict:
    pins = {"rmat": [], "pick_seeds": [], "frontiers": []}
    for scale, seed in ((6, 3), (7, 1), (8, 42), (8, 43), (10, 1), (12, 9)):
        src, dst = R.rmat_generate(scale, rng_seed=seed)
        pins["rmat"].append({"scale": scale, "rng_seed": seed, "m": int(len(src)),
                             "head": [[int(a), int(b)] for a, b in zip(src[:16], dst[:16])],
                             "sha256": sha(src, dst)})
    for scale, gseed, n, sseed in ((7, 1, 50, 9), (7, 1, 50, 10), (10, 4, 300, 1), (12, 2, 300, 7)):
        src, dst = R.rmat_generate(scale, rng_seed=gseed)
        g = R.build_bench_graph(src, dst, 1 << scale)
        pins["pick_seeds"].append({"scale": scale, "rng_seed": gseed, "n": n, "seed_rng": sseed,
                                   "seeds": [int(s) for s in g.pick_seeds(n, sseed)]})
    src, dst = R.rmat_generate(9, rng_seed=17)
    g = R.build_bench_graph(src, dst, 1 << 9)
    for s in g.pick_seeds(6, 17):
        for k in (1, 2, 3):
            for mode in (0, 1):
                pins["frontiers"].append({"scale": 9, "rng_seed": 17, "seed": int(s), "k": k,
                                          "mode": mode,
                                          "ids": [int(x) for x in g.k_hop_frontier(int(s), k, mode)]})
    # pick_seeds failure message (test_bench.cpp:104-113)
    g = R.build_bench_graph(np.array([0], np.uint32), np.array([1], np.uint32), 3)
    try:
        g.pick_seeds(2, 1)
        msg = None
    except oracle.RefError as e:
        msg = str(e)
    pins["pick_seeds_error"] = {"edges": [[0, 1]], "node_count": 3, "n": 2, "error": msg,
                                "ok_seeds": [int(s) for s in g.pick_seeds(1, 1)]}
    return pins


def walk_pins(R: oracle.Ref) -> dict:
    """walk_targets (execute.cpp:43-60) through the reference's Cypher executor:
    MATCH (a {id: S})-[*min..max]->(b) RETURN count(b) / RETURN b."""
    ranges = ((1, 1), (1, 2), (2, 2), (1, 3), (2, 4), (3, 3), (3, 6), (1, 32))
    out = {"ranges": [list(r) for r in ranges], "graphs": []}
    for scale, rng in ((6, 3), (7, 8), (8, 2), (9, 17)):
        src, dst = R.rmat_generate(scale, rng_seed=rng)
        g = R.build_bench_graph(src, dst, 1 << scale)
        seeds = [int(s) for s in g.pick_seeds(6, rng)]
        cases = []
        for s in seeds:
            for lo, hi in ranges:
                cnt = g.cypher(f"MATCH (a {{id: {s}}})-[*{lo}..{hi}]->(b) RETURN count(b)")
                ids = g.cypher(f"MATCH (a {{id: {s}}})-[*{lo}..{hi}]->(b) RETURN b")
                cases.append({"seed": s, "min": lo, "max": hi, "count": int(cnt.split("\n")[1]),
                              "ids": [int(t[1:]) for t in ids.split("\n")[1:] if t]})
        out["graphs"].append({"scale": scale, "rng_seed": rng, "cases": cases})
    # the seed reappears on a cycle; a self-loop keeps a walk alive (test_execute.cpp:89-97)
    edges = [[0, 1], [1, 2], [2, 0], [1, 1], [2, 3]]
    g = R.build_bench_graph(np.array([e[0] for e in edges], np.uint32),
                            np.array([e[1] for e in edges], np.uint32), 4)
    tl = []
    for s in range(4):
        for lo, hi in ((1, 1), (1, 3), (2, 2), (3, 3), (2, 5)):
            ids = g.cypher(f"MATCH (a {{id: {s}}})-[*{lo}..{hi}]->(b) RETURN b")
            tl.append({"seed": s, "min": lo, "max": hi,
                       "ids": [int(t[1:]) for t in ids.split("\n")[1:] if t]})
    out["cycle_loop"] = {"edges": edges, "node_count": 4, "cases": tl}
    return out


def main() -> None:
    R = oracle.Ref()
    for name, fn in (("known_answers", known_answers), ("c1_sweep", c1_sweep),
                     ("harness_pins", harness_pins), ("walk_pins", walk_pins)):
        data = fn(R)
        data["_generated_by"] = "tests/golden/make_golden.py from oracle/_ref (reference core)"
        (OUT / f"{name}.json").write_text(json.dumps(data, separators=(",", ":")) + "\n")
        print("wrote", name)


if __name__ == "__main__":
    main()

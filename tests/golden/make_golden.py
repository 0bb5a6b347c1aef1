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
* snapshot_pins.json — GRAPHSNAP1 texts (snapshot.cpp) parsed by the
  reference's snapshot_from_string: node count and relation CSRs of valid
  texts (some written by the reference's own snapshot_to_string), and the
  exact SnapshotError message of malformed ones.
* mxm_pins.json — mxm (sparse.cpp:292-363) over the three semirings, with
  and without masks: hand examples (test_sparse.cpp:165-243 shapes), a seeded
  random sweep of small matrices, RMAT graph products (SHA-256 of the result),
  and the dimension error texts.
* walk_pins.json — walk_targets (execute.cpp:43-60, the VarLenTraverse step)
  through the reference's own Cypher executor: counts and ids of
  MATCH (a {id: S})-[*min..max]->(b) and of the reversed pattern
  (a)<-[*min..max]-(b) (over transposed_matrix) on RMAT graphs and a cycle
  with a loop.

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
                # the reversed pattern walks the transpose (execute.cpp:35-39)
                in_ids = g.cypher(f"MATCH (a {{id: {s}}})<-[*{lo}..{hi}]-(b) RETURN b")
                cases.append({"seed": s, "min": lo, "max": hi, "count": int(cnt.split("\n")[1]),
                              "ids": [int(t[1:]) for t in ids.split("\n")[1:] if t],
                              "in_ids": [int(t[1:]) for t in in_ids.split("\n")[1:] if t]})
        out["graphs"].append({"scale": scale, "rng_seed": rng, "cases": cases})
    # the seed reappears on a cycle; a self-loop keeps a walk alive (test_execute.cpp:89-97)
    edges = [[0, 1], [1, 2], [2, 0], [1, 1], [2, 3]]
    g = R.build_bench_graph(np.array([e[0] for e in edges], np.uint32),
                            np.array([e[1] for e in edges], np.uint32), 4)
    tl = []
    for s in range(4):
        for lo, hi in ((1, 1), (1, 3), (2, 2), (3, 3), (2, 5)):
            ids = g.cypher(f"MATCH (a {{id: {s}}})-[*{lo}..{hi}]->(b) RETURN b")
            in_ids = g.cypher(f"MATCH (a {{id: {s}}})<-[*{lo}..{hi}]-(b) RETURN b")
            tl.append({"seed": s, "min": lo, "max": hi,
                       "ids": [int(t[1:]) for t in ids.split("\n")[1:] if t],
                       "in_ids": [int(t[1:]) for t in in_ids.split("\n")[1:] if t]})
    out["cycle_loop"] = {"edges": edges, "node_count": 4, "cases": tl}
    return out


def snapshot_pins(R: oracle.Ref) -> dict:
    """GRAPHSNAP1 (snapshot.cpp:127-231) through the reference parser/writer."""
    def csrs(g, rels):
        out = {}
        for r in rels:
            rp, ci = g.relation_csr(r)
            out["ANY" if r is None else r] = {"row_ptr": [int(x) for x in rp], "col_idx": [int(x) for x in ci]}
        return out

    valid, errors = [], []
    # 1. written by the reference: labels, every property type, two relations,
    #    a re-created edge (props overwritten), a self-loop
    g = R.graph(4)
    g.create_node("Person", "name:s:Ann%20Lee;age:i:31;score:f:1.5")
    g.create_node("Person,Admin", "ok:b:true;w:f:-0.25")
    g.create_node("", "")
    g.create_node("City", "big:f:1e10;t:s:a%3Bb%3Ac%25")
    g.create_node("", "inf:f:inf")
    for e in ((0, "KNOWS", 1, ""), (1, "KNOWS", 2, "since:i:2001"), (2, "LIKES", 0, ""), (0, "LIKES", 3, "w:f:0.5"),
              (3, "KNOWS", 3, ""), (1, "KNOWS", 2, "since:i:2002"), (4, "LIKES", 1, "")):
        g.create_edge(*e)
    t1 = g.snapshot()
    rels = [None, "KNOWS", "LIKES", "NOPE"]
    valid.append({"name": "writer_props_labels", "text": t1.decode(), "node_count": 5,
                  "csr": csrs(R.snapshot_parse(t1), rels)})
    # 2. hand-written: non-canonical order, duplicate lines, exotic literals the
    #    GPU fast path leaves to the host, blank trailing lines, no final newline
    t2 = ("GRAPHSNAP1\nNODES 6\n0\t\tx:f:.5\n1\tA\t\n2\t\ty:f:5.;z:i:-0\n3\t\t\n4\t\tq:s:\n5\t\t\n"
          "EDGES 9\n5\tR\t0\t\n0\tS\t1\t\n0\tR\t1\t\n0\tR\t1\tw:f:INF\n3\tR\t3\t\n2\tS\t4\tk:b:false\n"
          "4\tR\t2\t\n1\tR\t0\tk:i:-9223372036854775808\n0000002\tS\t0005\t\n\n\n").encode()
    valid.append({"name": "hand_unordered", "text": t2.decode(), "node_count": 6,
                  "csr": csrs(R.snapshot_parse(t2), [None, "R", "S", "T"])})
    t3 = b"GRAPHSNAP1\nNODES 0\nEDGES 0"
    valid.append({"name": "empty_graph", "text": t3.decode(), "node_count": 0,
                  "csr": csrs(R.snapshot_parse(t3), [None])})
    t4 = b"GRAPHSNAP1\nNODES 20\n" + b"".join(b"%d\t\t\n" % i for i in range(20)) + b"EDGES 2\n19\tE\t0\t\n0\tE\t19\t"
    valid.append({"name": "no_final_newline", "text": t4.decode(), "node_count": 20,
                  "csr": csrs(R.snapshot_parse(t4), [None, "E"])})
    # 3. a bench graph written by the reference (scale 9 RMAT, "EDGE" + ANY)
    src, dst = R.rmat_generate(9, rng_seed=5)
    bg = R.build_bench_graph(src, dst, 1 << 9)
    tb = bg.snapshot()
    pg = R.snapshot_parse(tb)
    rp, ci = pg.relation_csr(None)
    bench = {"scale": 9, "rng_seed": 5, "text_sha256": hashlib.sha256(tb).hexdigest(), "bytes": len(tb),
             "node_count": pg.node_count, "any_csr_sha256": sha(rp, ci),
             "edge_csr_sha256": sha(*pg.relation_csr("EDGE")),
             "counts_k2": [pg.k_hop_count(int(s), 2) for s in pg.pick_seeds(8, 1)],
             "seeds": [int(s) for s in pg.pick_seeds(8, 1)]}
    # 4. malformed texts: the reference's exact message
    H = b"GRAPHSNAP1\nNODES 3\n0\t\t\n1\tA,B\tx:i:5\n2\t\t\n"
    bad = {
        "empty": b"", "header_crlf": H.replace(b"\n", b"\r\n") + b"EDGES 0\r\n",
        "header_space": b"GRAPHSNAP1 \nNODES 0\nEDGES 0\n", "no_nodes_line": b"GRAPHSNAP1",
        "nodes_word": b"GRAPHSNAP1\nNODE 3\n", "nodes_plus": b"GRAPHSNAP1\nNODES +1\n0\t\t\nEDGES 0\n",
        "nodes_huge": b"GRAPHSNAP1\nNODES 99999999999999999999\n",
        "nodes_eof": b"GRAPHSNAP1\nNODES 3\n0\t\t\n", "node_fields": b"GRAPHSNAP1\nNODES 1\n0\t\nEDGES 0\n",
        "node_id_bad": b"GRAPHSNAP1\nNODES 1\nx\t\t\nEDGES 0\n",
        "node_id_order": b"GRAPHSNAP1\nNODES 2\n0\t\t\n0\t\t\nEDGES 0\n",
        "label_empty": b"GRAPHSNAP1\nNODES 1\n0\tA,\t\nEDGES 0\n",
        "label_digit": b"GRAPHSNAP1\nNODES 1\n0\t1A\tq\nEDGES 0\n",
        "label_bad_props_ok": b"GRAPHSNAP1\nNODES 1\n0\tA-B\tk:i:1\nEDGES 0\n",
        "no_edges_line": H, "edges_word": H + b"EDGE 1\n", "edges_count": H + b"EDGES x\n",
        "edges_eof": H + b"EDGES 3\n0\tR\t1\t\n", "edge_fields": H + b"EDGES 1\n0\tR\t1\n",
        "edge_fields5": H + b"EDGES 1\n0\tR\t1\t\t\n",
        "edge_src_props": H + b"EDGES 1\nx\tR\t1\tq\n", "edge_src_dst": H + b"EDGES 1\nx\tR\ty\t\n",
        "edge_range_rel": H + b"EDGES 1\n9\t1R\t1\t\n", "edge_dst_range": H + b"EDGES 1\n0\tR\t3\t\n",
        "edge_rel_bad": H + b"EDGES 1\n0\tR-S\t1\t\n", "edge_rel_empty": H + b"EDGES 1\n0\t\t1\t\n",
        "edge_later_line": H + b"EDGES 3\n0\tR\t1\t\n1\tR\t2\t\n2\tR\t0\tk:b:yes\n",
        "trailing": H + b"EDGES 0\n\nx\n",
        "item_short": H.replace(b"x:i:5", b"x:i") + b"EDGES 0\n",
        "item_empty_value": H.replace(b"x:i:5", b"x:i:") + b"EDGES 0\n",
        "item_empty": H.replace(b"x:i:5", b"x:i:5;") + b"EDGES 0\n",
        "item_nocolon": H.replace(b"x:i:5", b"abc") + b"EDGES 0\n",
        "item_double_colon": H.replace(b"x:i:5", b"x::5") + b"EDGES 0\n",
        "key_bad": H.replace(b"x:i:5", b"1x:i:5") + b"EDGES 0\n",
        "type_bad": H.replace(b"x:i:5", b"x:z:1") + b"EDGES 0\n",
        "int_plus": H.replace(b"x:i:5", b"x:i:+5") + b"EDGES 0\n",
        "int_space": H.replace(b"x:i:5", b"x:i: 5") + b"EDGES 0\n",
        "int_overflow": H.replace(b"x:i:5", b"x:i:9223372036854775808") + b"EDGES 0\n",
        "float_plus": H.replace(b"x:i:5", b"x:f:+5") + b"EDGES 0\n",
        "float_hex": H.replace(b"x:i:5", b"x:f:0x1p3") + b"EDGES 0\n",
        "float_big": H.replace(b"x:i:5", b"x:f:1e400") + b"EDGES 0\n",
        "float_tiny": H.replace(b"x:i:5", b"x:f:1e-400") + b"EDGES 0\n",
        "float_exp": H.replace(b"x:i:5", b"x:f:5e") + b"EDGES 0\n",
        "bool_case": H.replace(b"x:i:5", b"x:b:True") + b"EDGES 0\n",
        "pct_trunc": H.replace(b"x:i:5", b"x:s:a%2") + b"EDGES 0\n",
        "pct_trunc0": H.replace(b"x:i:5", b"x:s:%") + b"EDGES 0\n",
        "pct_bad": H.replace(b"x:i:5", b"x:s:a%zz") + b"EDGES 0\n",
        "two_errors_first_wins": H.replace(b"x:i:5", b"x:f:+1") + b"EDGES 1\nx\tR\t1\t\n",
    }
    for name, text in bad.items():
        try:
            R.snapshot_parse(text)
            raise SystemExit(f"snapshot case {name} unexpectedly parsed")
        except oracle.RefError as e:
            errors.append({"name": name, "text": text.decode(), "error": str(e)})
    return {"valid": valid, "bench": bench, "errors": errors}


def mxm_pins(R: oracle.Ref) -> dict:
    """mxm through the reference (from_parts operands, vals None = structural)."""
    def enc(m):
        nr, nc, rp, ci, v = m
        return {"nrows": int(nr), "ncols": int(nc), "row_ptr": [int(x) for x in rp],
                "col_idx": [int(x) for x in ci], "vals": None if v is None else [int(x) for x in v]}

    def from_dense(p, v, valued):
        nr, nc = p.shape
        rp = [0]
        ci, vals = [], []
        for i in range(nr):
            for j in range(nc):
                if p[i, j]:
                    ci.append(j)
                    vals.append(int(v[i, j]))
            rp.append(len(ci))
        return (nr, nc, np.array(rp, np.uint64), np.array(ci, np.uint64),
                np.array(vals, np.int64) if valued else None)

    cases = []

    def add(name, a, b, sr, mask=None):
        c = R.mxm(a, b, sr, mask)
        cases.append({"name": name, "semiring": sr, "a": enc(a), "b": enc(b),
                      "mask": None if mask is None else enc(mask), "c": enc(c)})

    path = (4, 4, np.array([0, 1, 2, 3, 3], np.uint64), np.array([1, 2, 3], np.uint64), None)
    add("path_squared", path, path, 0)
    add("path_squared_masked", path, path, 0, (4, 4, np.array([0, 1, 1, 1, 1]), np.array([2]), None))
    add("plus_times_2x2", (2, 2, np.array([0, 2, 3]), np.array([0, 1, 1]), np.array([1, 2, 3])),
        (2, 2, np.array([0, 1, 3]), np.array([0, 0, 1]), np.array([4, 5, 6])), 1)
    add("min_plus_3x3", (3, 3, np.array([0, 2, 3, 3]), np.array([1, 2, 2]), np.array([5, 9, 2])),
        (3, 3, np.array([0, 2, 3, 3]), np.array([1, 2, 2]), np.array([5, 9, 2])), 2)
    pat = (3, 3, np.array([0, 1, 2, 2]), np.array([1, 2]), None)
    add("structural_plus_times", pat, pat, 1)
    add("empty_valued", (2, 2, np.array([0, 0, 0]), np.array([]), np.array([], np.int64)),
        (2, 2, np.array([0, 1, 1]), np.array([0]), np.array([3])), 1)
    add("wraparound", (1, 1, np.array([0, 1]), np.array([0]), np.array([2 ** 62])),
        (1, 2, np.array([0, 2]), np.array([0, 1]), np.array([4, -(2 ** 63)])), 1)
    rng = np.random.default_rng(202)
    for trial in range(150):
        m, k, n = (int(x) for x in rng.integers(1, 21, 3))
        sr = trial % 3
        dens = (0.02, 0.1, 0.35)[(trial // 3) % 3]
        valued = sr != 0
        pa = rng.random((m, k)) < dens
        pb = rng.random((k, n)) < dens
        va = rng.integers(-50, 50, (m, k))
        vb = rng.integers(-50, 50, (k, n))
        mask = None
        if trial % 4 == 0:
            pm = rng.random((m, n)) < 0.5
            mask = from_dense(pm, pm, False)
        add(f"random_{trial}", from_dense(pa, va, valued), from_dense(pb, vb, valued), sr, mask)
    out = {"cases": cases, "graphs": []}
    for scale, rng_seed in ((9, 2), (10, 7)):
        src, dst = R.rmat_generate(scale, rng_seed=rng_seed)
        g = R.build_bench_graph(src, dst, 1 << scale)
        rp, ci = g.relation_csr(None)
        A = (len(rp) - 1, len(rp) - 1, rp, ci, None)
        ent = {"scale": scale, "rng_seed": rng_seed}
        for key, sr, mask in (("bool", 0, None), ("plus_times", 1, None), ("min_plus", 2, None),
                              ("bool_masked_by_A", 0, A)):
            c = R.mxm(A, A, sr, mask)
            ent[key] = {"nnz": int(len(c[3])),
                        "sha256": sha(c[2], c[3], c[4] if c[4] is not None else np.zeros(0, np.int64))}
        out["graphs"].append(ent)
    errs = []
    for a, b, mask in (((2, 3), (4, 2), None), ((5, 4), (4, 6), (5, 5)), ((3, 3), (3, 3), (2, 3))):
        A = (a[0], a[1], np.zeros(a[0] + 1, np.uint64), np.zeros(0, np.uint64), None)
        B = (b[0], b[1], np.zeros(b[0] + 1, np.uint64), np.zeros(0, np.uint64), None)
        M = None if mask is None else (mask[0], mask[1], np.zeros(mask[0] + 1, np.uint64), np.zeros(0, np.uint64), None)
        try:
            R.mxm(A, B, 0, M)
            raise SystemExit("mxm dimension case unexpectedly passed")
        except oracle.RefError as e:
            errs.append({"a": list(a), "b": list(b), "mask": None if mask is None else list(mask), "error": str(e)})
    out["errors"] = errs
    return out


def main() -> None:
    R = oracle.Ref()
    for name, fn in (("known_answers", known_answers), ("c1_sweep", c1_sweep),
                     ("harness_pins", harness_pins), ("walk_pins", walk_pins),
                     ("snapshot_pins", snapshot_pins), ("mxm_pins", mxm_pins)):
        data = fn(R)
        data["_generated_by"] = "tests/golden/make_golden.py from oracle/_ref (reference core)"
        (OUT / f"{name}.json").write_text(json.dumps(data, separators=(",", ":")) + "\n")
        print("wrote", name)


if __name__ == "__main__":
    main()

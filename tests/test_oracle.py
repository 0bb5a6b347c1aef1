"""The CPU oracle (oracle/khop_oracle.c) pinned against the reference's own
outputs (tests/golden/*.json, generated from oracle/_ref by make_golden.py)."""
import hashlib

import numpy as np
import pytest

import oracle


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def test_rmat_pins(port, pins):
    for p in pins["rmat"]:
        src, dst = port.rmat_generate(p["scale"], rng_seed=p["rng_seed"])
        assert len(src) == p["m"]
        assert [[int(a), int(b)] for a, b in zip(src[:16], dst[:16])] == p["head"]
        assert sha(src, dst) == p["sha256"]


def test_pick_seeds_pins(port, pins):
    for p in pins["pick_seeds"]:
        src, dst = port.rmat_generate(p["scale"], rng_seed=p["rng_seed"])
        rp, _ = port.build_csr(1 << p["scale"], src, dst)
        assert port.pick_seeds(rp, p["n"], p["seed_rng"]).tolist() == p["seeds"]
    e = pins["pick_seeds_error"]
    rp, _ = port.build_csr(e["node_count"], np.array([0], np.uint32), np.array([1], np.uint32))
    assert port.pick_seeds(rp, 1, 1).tolist() == e["ok_seeds"]
    with pytest.raises(RuntimeError, match="need 2 seeds but only 1 nodes have out-degree >= 1"):
        port.pick_seeds(rp, 2, 1)
    assert e["error"] == "need 2 seeds but only 1 nodes have out-degree >= 1"


def test_known_answers(port, known):
    for case in known["cases"]:
        g = known[case["graph"]]
        rp = np.array(g["row_ptr"], np.uint64)
        ci = np.array(g["col_idx"], np.uint64)
        got = port.khop_frontier(rp, ci, case["seed"], case["k"], case["mode"])
        assert got.tolist() == case["frontier"], case
        assert len(got) == case["count"]
    # the literal pins of proj/tests/test_execute.cpp:104-120
    p = {(c["graph"], c["seed"], c["k"], c["mode"]): c for c in known["cases"]}
    assert p[("path4", 0, 2, 0)]["count"] == 1 and p[("path4", 0, 2, 0)]["frontier"] == [2]
    assert p[("path4", 3, 1, 0)]["count"] == 0
    assert p[("path4", 0, 6, 1)]["count"] == 3
    assert p[("triangle", 0, 3, 0)]["count"] == 0
    assert p[("triangle", 0, 3, 1)]["count"] == 2


def test_relation_filter_pins(known):
    r = known["relation_filter"]  # test_execute.cpp:122-129
    assert r["R"]["count_seed0_k1"] == 1
    assert r["ANY"]["count_seed0_k1"] == 2
    assert r["S"]["count_seed0_k1"] == 1
    assert r["NONE"]["count_seed0_k1"] == 0


def test_c1_sweep(port, c1):
    """acceptance c1 (8000 counts) reproduced by both oracle functions."""
    total = 0
    for g in c1["graphs"]:
        src, dst = port.rmat_generate(g["scale"], rng_seed=g["rng_seed"])
        assert sha(src, dst) == g["edges_sha256"]
        n = g["node_count"]
        rp, ci = port.build_csr(n, src, dst)
        assert sha(rp, ci) == g["csr_sha256"]
        assert port.pick_seeds(rp, 50, g["rng_seed"]).tolist() == g["seeds"]
        adj = port.bfs_oracle(n, src, dst)
        for mode in (0, 1):
            for k in c1["ks"]:
                want = g["counts"][f"{mode}_{k}"]
                got_bfs = [adj.count(s, k, mode) for s in g["seeds"]]
                got_vxm = [port.khop_count(rp, ci, s, k, mode) for s in g["seeds"]]
                assert got_bfs == want and got_vxm == want
                total += len(want)
    assert total == 8000


def test_frontier_pins(port, pins):
    src, dst = port.rmat_generate(9, rng_seed=17)
    rp, ci = port.build_csr(1 << 9, src, dst)
    for f in pins["frontiers"]:
        assert port.khop_frontier(rp, ci, f["seed"], f["k"], f["mode"]).tolist() == f["ids"]


def test_work_model(port):
    """E(s,k) and level sizes agree with the frontier sets."""
    src, dst = port.rmat_generate(10, rng_seed=4)
    rp, ci = port.build_csr(1 << 10, src, dst)
    for s in port.pick_seeds(rp, 20, 3):
        e, sizes = port.khop_work(rp, ci, int(s), 6)
        for k in range(1, len(sizes)):
            assert sizes[k] == port.khop_count(rp, ci, int(s), k, 0)
        deg = np.diff(rp.astype(np.int64))
        fr = [np.array([s])] + [port.khop_frontier(rp, ci, int(s), k, 0) for k in range(1, len(sizes))]
        expanded = len(sizes) - 1
        assert e == sum(int(deg[f.astype(np.int64)].sum()) for f in fr[:expanded])


@pytest.mark.skipif(not oracle.REF_SO.exists(), reason="reference not built here")
def test_port_matches_reference_library(port):
    R = oracle.Ref()
    src, dst = R.rmat_generate(11, rng_seed=77)
    g = R.build_bench_graph(src, dst, 1 << 11)
    rp, ci = g.relation_csr()
    for s in g.pick_seeds(25, 77):
        for k in (1, 2, 3, 6, 32):
            for mode in (0, 1):
                assert port.khop_count(rp, ci, int(s), k, mode) == g.k_hop_count(int(s), k, mode)


def test_walk_pins(port):
    """walk_targets restated (oracle) vs the reference's Cypher executor."""
    from conftest import load_golden
    w = load_golden("walk_pins")
    for gd in w["graphs"]:
        src, dst = port.rmat_generate(gd["scale"], rng_seed=gd["rng_seed"])
        rp, ci = port.build_csr(1 << gd["scale"], src, dst)
        for c in gd["cases"]:
            got = port.walk_targets(rp, ci, c["seed"], c["min"], c["max"])
            assert got.tolist() == c["ids"] and len(got) == c["count"], c
    cl = w["cycle_loop"]
    e = np.array(cl["edges"], np.uint32)
    rp, ci = port.build_csr(cl["node_count"], e[:, 0], e[:, 1])
    for c in cl["cases"]:
        assert port.walk_targets(rp, ci, c["seed"], c["min"], c["max"]).tolist() == c["ids"], c

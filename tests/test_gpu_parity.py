"""Bit-exact parity of the sm_100a k-hop kernels (through the C ABI) against
the reference's golden vectors and the CPU oracle.

Every test here runs the product path: libmgk.so's SINGLE and LANES engines.
The oracle (oracle/) is only the checker."""
import hashlib

import numpy as np
import pytest

from paper_1905_01294_b200 import (ENGINE_LANES, ENGINE_SINGLE, ContractError, DeviceGraph,
                                   KHopQuery, TraverseMode, Tuning, harness as H, k_hop_count,
                                   k_hop_count_batch, k_hop_frontier)

pytestmark = pytest.mark.gpu
KS = (1, 2, 3, 6)


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def graph_of(g):
    return DeviceGraph.from_csr(np.array(g["row_ptr"], np.uint64), np.array(g["col_idx"], np.uint64),
                                node_count=g.get("node_count"))


# ---- known answers (proj/tests/test_execute.cpp:104-139) ---------------------------
def test_known_answers(known):
    graphs = {name: graph_of({**known[name], "node_count": known[name]["node_count"]})
              for name in ("path4", "triangle")}
    for case in known["cases"]:
        g = graphs[case["graph"]]
        q = KHopQuery(case["seed"], case["k"], TraverseMode(case["mode"]))
        assert k_hop_count(g, q) == case["count"], case
        assert k_hop_frontier(g, q).tolist() == case["frontier"], case
        for eng in (ENGINE_SINGLE, ENGINE_LANES):
            got = k_hop_count_batch(g, [case["seed"]], case["k"], case["mode"], engine=eng)
            assert int(got[0]) == case["count"], (case, eng)


def test_relation_filter(known):
    for rel, want in (("R", 1), ("ANY", 2), ("S", 1), ("NONE", 0)):
        r = known["relation_filter"][rel]
        g = DeviceGraph.from_csr(np.array(r["row_ptr"], np.uint64), np.array(r["col_idx"], np.uint64),
                                 node_count=4)
        assert k_hop_count(g, KHopQuery(0, 1)) == want == r["count_seed0_k1"]


def test_error_strings(known):
    p = known["path4"]
    g = DeviceGraph.from_csr(np.array(p["row_ptr"], np.uint64), np.array(p["col_idx"], np.uint64),
                             node_count=p["node_count"])
    for e in known["errors"]:
        with pytest.raises(ContractError) as ex:
            k_hop_count(g, KHopQuery(e["seed"], e["k"]))
        assert str(ex.value) == e["error"]
    # the C ABI itself checks against the matrix dimension with the same text
    with pytest.raises(ContractError, match="k-hop seed 99 is not an allocated node"):
        g.node_count = 10 ** 6
        k_hop_count_batch(g, [99], 1)
    with pytest.raises(ContractError, match=r"k-hop count 33 outside \[1, 32\]"):
        k_hop_count_batch(g, [0], 33)


# ---- acceptance c1: 8000 golden counts ------------------------------------------------
@pytest.mark.parametrize("engine", [ENGINE_SINGLE, ENGINE_LANES])
def test_c1_sweep(port, c1, engine):
    total = 0
    for gd in c1["graphs"]:
        src, dst = port.rmat_generate(gd["scale"], rng_seed=gd["rng_seed"])
        assert sha(src, dst) == gd["edges_sha256"]
        n = gd["node_count"]
        # device-side build (sort + dedup + CSR/CSC) must equal the reference's flush
        g = DeviceGraph.from_edges(src, dst, n)
        rp, ci = g.csr()
        assert sha(rp.astype(np.uint64), ci.astype(np.uint64)) == gd["csr_sha256"]
        seeds = np.array(gd["seeds"], np.uint64)
        for mode in (0, 1):
            for k in c1["ks"]:
                got = k_hop_count_batch(g, seeds, k, mode, engine=engine)
                assert got.tolist() == gd["counts"][f"{mode}_{k}"], (gd["rng_seed"], mode, k)
                total += len(seeds)
    assert total == 8000


def test_frontier_pins(port, pins):
    src, dst = port.rmat_generate(9, rng_seed=17)
    g = DeviceGraph.from_edges(src, dst, 1 << 9)
    for f in pins["frontiers"]:
        got = k_hop_frontier(g, KHopQuery(f["seed"], f["k"], TraverseMode(f["mode"])))
        assert got.tolist() == f["ids"]


@pytest.mark.parametrize("via", ["edges", "csr"])
def test_csc_is_transpose(port, via):
    """CSC = transpose (sparse.cpp:379-403) as sets per column; each in-list is
    ordered by descending out-degree of the in-neighbour (ties ascending id)."""
    src, dst = port.rmat_generate(10, rng_seed=3)
    n = 1 << 10
    g = DeviceGraph.from_edges(src, dst, n)
    rp, ci = g.csr()
    if via == "csr":
        g = DeviceGraph.from_csr(rp, ci)
    cp, ri = g.csc()
    trp, tci = port.build_csr(n, ci, H.csr_to_edges(rp, ci)[0])
    assert (cp == trp).all()
    deg = np.diff(rp.astype(np.int64))
    for c in range(n):
        seg = ri[cp[c]:cp[c + 1]].astype(np.int64)
        assert sorted(seg.tolist()) == tci[trp[c]:trp[c + 1]].tolist()
        want = sorted(seg.tolist(), key=lambda r: (-deg[r], r))
        assert seg.tolist() == want


# ---- config 1 (scale 16, 300 seeds) and direction/lane variants ----------------------------
@pytest.fixture(scope="module")
def g1():
    rp, ci = H.gen_csr(H.G1)
    return rp, ci, DeviceGraph.from_csr(rp, ci)


def oracle_counts(port, rp, ci, seeds, k, mode):
    rp64, ci64 = rp.astype(np.uint64), ci.astype(np.uint64)
    return [port.khop_count(rp64, ci64, int(s), k, mode) for s in seeds]


def test_cfg1_parity(port, g1):
    rp, ci, g = g1
    seeds = H.pick_seeds(rp, 300, 1)
    for mode in (0, 1):
        for k in KS:
            want = oracle_counts(port, rp, ci, seeds, k, mode)
            for eng in (ENGINE_LANES, ENGINE_SINGLE):
                assert k_hop_count_batch(g, seeds, k, mode, engine=eng).tolist() == want, (mode, k, eng)


@pytest.mark.parametrize("force", [1, 2])
@pytest.mark.parametrize("words", [1, 2, 4, 8])
def test_directions_and_lane_widths(port, g1, force, words):
    rp, ci, g = g1
    seeds = H.pick_seeds(rp, 200, 7)
    want = {(k, m): oracle_counts(port, rp, ci, seeds, k, m) for k in (2, 3, 6) for m in (0, 1)}
    try:
        g.set_tuning(Tuning(force_dir=force, lanes_words=words))
        for (k, m), w in want.items():
            assert k_hop_count_batch(g, seeds, k, m, engine=ENGINE_LANES).tolist() == w, (k, m)
            if words == 1:
                assert k_hop_count_batch(g, seeds[:12], k, m, engine=ENGINE_SINGLE).tolist() == w[:12]
    finally:
        g.set_tuning(Tuning())


@pytest.mark.parametrize("force", [0, 1, 2])
def test_narrow_lane_words(port, g1, force, monkeypatch):
    """Batches of <= 8 / 10 / 16 seeds use 8-bit, 10-bit (three per 32-bit
    word, atomics for every write) and 16-bit lane words; each width, forced
    with MGK_LANE_BITS, and the 64-bit words give the oracle's counts."""
    rp, ci, g = g1
    seeds = H.pick_seeds(rp, 60, 11)
    groups = [seeds[0:10], seeds[10:20], seeds[20:29], seeds[29:37], seeds[37:38]]
    want = {(j, k, m): oracle_counts(port, rp, ci, grp, k, m)
            for j, grp in enumerate(groups) for k in (1, 2, 3, 6) for m in (0, 1)}
    try:
        g.set_tuning(Tuning(force_dir=force))
        for bits in ("8", "10", "16", "64"):
            monkeypatch.setenv("MGK_LANE_BITS", bits)
            for (j, k, m), w in want.items():
                got = k_hop_count_batch(g, groups[j], k, m, engine=ENGINE_LANES).tolist()
                assert got == w, (bits, j, k, m)
    finally:
        g.set_tuning(Tuning())


def test_duplicate_and_isolated_seeds(port, g1):
    rp, ci, g = g1
    deg = np.diff(rp.astype(np.int64))
    iso = np.flatnonzero(deg == 0)[:3]
    seeds = np.array(list(H.pick_seeds(rp, 5, 3)) * 3 + list(iso), np.uint64)
    for k in (1, 3):
        for m in (0, 1):
            want = oracle_counts(port, rp, ci, seeds, k, m)
            for eng in (ENGINE_LANES, ENGINE_SINGLE):
                assert k_hop_count_batch(g, seeds, k, m, engine=eng).tolist() == want


def test_empty_batch_and_empty_graph():
    g = DeviceGraph.from_csr(np.zeros(5, np.uint32), np.zeros(0, np.uint32))
    assert k_hop_count_batch(g, [], 2).tolist() == []
    assert k_hop_count_batch(g, [0, 3], 2, 1).tolist() == [0, 0]
    assert k_hop_frontier(g, KHopQuery(1, 1, TraverseMode.Cumulative)).tolist() == []


def test_many_batches_stats(port, g1):
    rp, ci, g = g1
    seeds = H.pick_seeds(rp, 1500, 11)
    counts, st = k_hop_count_batch(g, seeds, 2, 0, engine=ENGINE_LANES, stats=True)
    want = oracle_counts(port, rp, ci, seeds, 2, 0)
    assert counts.tolist() == want
    assert st["levels"][2]["frontier"] == sum(want)
    e = sum(port.khop_work(rp.astype(np.uint64), ci.astype(np.uint64), int(s), 2)[0] for s in seeds)
    assert st["levels"][1]["edges"] + st["levels"][2]["edges"] == e


# ---- config 2 graph at full size ------------------------------------------------------
@pytest.fixture(scope="module")
def g2():
    rp, ci = H.gen_csr(H.G2)
    return rp, ci, DeviceGraph.from_csr(rp, ci)


def test_g2_sampled_oracle(port, g2):
    rp, ci, g = g2
    seeds = H.pick_seeds(rp, 300, 1)
    for k in (1, 2):
        want = oracle_counts(port, rp, ci, seeds[:40], k, 0)
        assert k_hop_count_batch(g, seeds, k, 0)[:40].tolist() == want
    for k in (3, 6):
        want = oracle_counts(port, rp, ci, seeds[:3], k, 0)
        assert k_hop_count_batch(g, seeds[:10], k, 0)[:3].tolist() == want
        assert k_hop_count_batch(g, seeds[:3], k, 0, engine=ENGINE_SINGLE).tolist() == want


def test_g2_properties(g2):
    """Size-independent properties at full size: cumulative(k) = sum of exact(1..k);
    engines and lane widths agree; the 64-lane batches of a 65,536-seed run agree
    with a re-run in a different batch order."""
    rp, ci, g = g2
    seeds = H.pick_seeds(rp, 2048, 5)
    ex = [k_hop_count_batch(g, seeds, k, 0) for k in range(1, 7)]
    cum6 = k_hop_count_batch(g, seeds, 6, 1)
    assert (np.sum(ex, axis=0) == cum6).all()
    perm = np.random.default_rng(0).permutation(len(seeds))
    assert (k_hop_count_batch(g, seeds[perm], 3, 0) == ex[2][perm]).all()
    single = k_hop_count_batch(g, seeds[:4], 6, 1, engine=ENGINE_SINGLE)
    assert (single == cum6[:4]).all()


def test_g2_single_directions_at_depth(g2):
    """300 seeds x k=6 in the SINGLE engine: the push item lists overflow (the
    engine then pulls those seeds, even when push is forced) and every
    direction policy gives the same answers."""
    rp, ci, g = g2
    seeds = H.pick_seeds(rp, 300, 1)
    want = k_hop_count_batch(g, seeds, 6, 0, engine=ENGINE_LANES)
    try:
        for t in (Tuning(), Tuning(force_dir=1), Tuning(force_dir=2), Tuning(alpha=60, alpha_last=60)):
            g.set_tuning(t)
            assert (k_hop_count_batch(g, seeds, 6, 0, engine=ENGINE_SINGLE) == want).all(), t
    finally:
        g.set_tuning(Tuning())


@pytest.mark.parametrize("force", [0, 1, 2])
def test_frontier_ids_deep(port, g1, force):
    """k_hop_frontier's sorted ids (exact and cumulative) at depth, every direction."""
    rp, ci, g = g1
    rp64, ci64 = rp.astype(np.uint64), ci.astype(np.uint64)
    try:
        g.set_tuning(Tuning(force_dir=force))
        for s in H.pick_seeds(rp, 4, 21):
            for k in (2, 3, 4, 6):
                for mode in (0, 1):
                    want = port.khop_frontier(rp64, ci64, int(s), k, mode)
                    got = k_hop_frontier(g, KHopQuery(int(s), k, TraverseMode(mode)))
                    assert np.array_equal(got, want), (int(s), k, mode, force)
    finally:
        g.set_tuning(Tuning())


@pytest.mark.parametrize("spec", [
    H.GraphSpec("a", scale=10, edge_factor=8, target_unique=0, relabel=0, rng_seed=3),
    H.GraphSpec("b", scale=12, edge_factor=8, target_unique=20000, relabel=2, rng_seed=5),
    H.GraphSpec("c", scale=14, edge_factor=4, target_unique=0, relabel=1, rng_seed=9),
    H.G1,
], ids=lambda s: s.name)
def test_device_generator_equals_host(spec):
    """mgk_graph_gen_rmat (GPU) builds exactly the CSR of mgk_gen_rmat_csr (host)."""
    rp, ci = H.gen_csr(spec)
    g = DeviceGraph.generate(spec)
    drp, dci = g.csr()
    assert g.nrows == len(rp) - 1
    assert np.array_equal(drp, rp) and np.array_equal(dci, ci)


def test_device_generator_g2(g2):
    rp, ci, _ = g2
    g = DeviceGraph.generate(H.G2)
    drp, dci = g.csr()
    assert np.array_equal(drp, rp) and np.array_equal(dci, ci)


# ---- walk_targets (execute.cpp:43-60): the Cypher variable-length route -------------------
@pytest.mark.parametrize("engine", [ENGINE_SINGLE, ENGINE_LANES])
def test_walk_pins(port, engine):
    """Counts and ids of MATCH (a {id: S})-[*min..max]->(b) from the reference's
    own executor (tests/golden/walk_pins.json)."""
    from conftest import load_golden
    from paper_1905_01294_b200 import walk_count_batch, walk_targets
    w = load_golden("walk_pins")
    for gd in w["graphs"]:
        src, dst = port.rmat_generate(gd["scale"], rng_seed=gd["rng_seed"])
        g = DeviceGraph.from_edges(src, dst, 1 << gd["scale"])
        by_range = {}
        for c in gd["cases"]:
            by_range.setdefault((c["min"], c["max"]), []).append(c)
        for (lo, hi), cases in by_range.items():
            seeds = [c["seed"] for c in cases]
            got = walk_count_batch(g, seeds, lo, hi, engine=engine)
            assert got.tolist() == [c["count"] for c in cases], (lo, hi)
            if engine == ENGINE_SINGLE:
                for c in cases[:3]:
                    assert walk_targets(g, c["seed"], lo, hi).tolist() == c["ids"], c
    cl = w["cycle_loop"]
    e = np.array(cl["edges"], np.uint32)
    g = DeviceGraph.from_edges(e[:, 0], e[:, 1], cl["node_count"])
    for c in cl["cases"]:
        assert walk_count_batch(g, [c["seed"]], c["min"], c["max"], engine=engine).tolist() == [len(c["ids"])]
        assert walk_targets(g, c["seed"], c["min"], c["max"]).tolist() == c["ids"], c


def test_walk_cfg1_and_messages(port, g1):
    from paper_1905_01294_b200 import walk_count_batch, walk_targets
    rp, ci, g = g1
    rp64, ci64 = rp.astype(np.uint64), ci.astype(np.uint64)
    seeds = H.pick_seeds(rp, 64, 4)
    for lo, hi in ((1, 2), (2, 3), (3, 6), (1, 6)):
        want = [len(port.walk_targets(rp64, ci64, int(s), lo, hi)) for s in seeds]
        for eng in (ENGINE_SINGLE, ENGINE_LANES):
            assert walk_count_batch(g, seeds, lo, hi, engine=eng).tolist() == want, (lo, hi, eng)
        assert np.array_equal(walk_targets(g, int(seeds[0]), lo, hi),
                              port.walk_targets(rp64, ci64, int(seeds[0]), lo, hi))
    for (lo, hi), msg in (((0, 2), "hop minimum must be at least 1"),
                          ((1, 33), "hop count 33 exceeds the cap of 32"),
                          ((4, 2), "hop maximum 2 is less than minimum 4")):
        with pytest.raises(ContractError, match=msg):
            walk_count_batch(g, seeds[:1], lo, hi)


# ---- opt-in locality relabelling (MGK_RELABEL=1): ids stay external at the boundary -----
def test_relabelled_layout(port, g1, monkeypatch):
    """The in-degree relabelled device layout answers exactly like the
    external-id layout: counts (both engines, both modes), frontier and walk
    ids (mapped back and sorted), and the downloaded CSR / CSC."""
    from paper_1905_01294_b200 import walk_count_batch, walk_targets
    rp, ci, g0 = g1
    monkeypatch.setenv("MGK_RELABEL", "1")
    g = DeviceGraph.from_csr(rp, ci)
    monkeypatch.delenv("MGK_RELABEL")
    rp64, ci64 = rp.astype(np.uint64), ci.astype(np.uint64)
    drp, dci = g.csr()
    assert np.array_equal(drp, rp) and np.array_equal(dci, ci)
    cp0, ri0 = g0.csc()
    cp1, ri1 = g.csc()
    assert np.array_equal(cp0, cp1) and np.array_equal(ri0, ri1)
    seeds = H.pick_seeds(rp, 300, 11)
    for mode in (0, 1):
        for k in (1, 2, 3, 6):
            want = oracle_counts(port, rp, ci, seeds, k, mode)
            for eng in (ENGINE_SINGLE, ENGINE_LANES):
                assert k_hop_count_batch(g, seeds, k, mode, engine=eng).tolist() == want, (mode, k, eng)
    for s in seeds[:4]:
        for k, mode in ((1, 0), (2, 0), (3, 1)):
            want = port.khop_frontier(rp64, ci64, int(s), k, mode)
            assert np.array_equal(k_hop_frontier(g, KHopQuery(int(s), k, TraverseMode(mode))), want)
        assert np.array_equal(walk_targets(g, int(s), 2, 3), port.walk_targets(rp64, ci64, int(s), 2, 3))
    assert walk_count_batch(g, seeds[:50], 1, 3).tolist() == \
        [len(port.walk_targets(rp64, ci64, int(s), 1, 3)) for s in seeds[:50]]


# ---- multi-GPU entry: seed-sharded replicas ------------------------------
def test_replicas_and_multi(port, g1):
    """mgk_graph_replicate + mgk_khop_count_multi. This box has one GPU, so the
    replicas all live on device 0; the sharding, per-replica streams and
    threads are the same code a multi-GPU node runs."""
    from paper_1905_01294_b200 import k_hop_count_multi
    rp, ci, g = g1
    reps = [g, g.replicate(0), g.replicate(0)]
    drp, dci = reps[2].csr()
    assert np.array_equal(drp, rp) and np.array_equal(dci, ci)
    seeds = H.pick_seeds(rp, 301, 5)
    for k in (1, 2, 3):
        for mode in (0, 1):
            want = k_hop_count_batch(g, seeds, k, mode)
            assert want.tolist() == oracle_counts(port, rp, ci, seeds[:40], k, mode) + want.tolist()[40:]
            for nrep in (1, 2, 3):
                assert k_hop_count_multi(reps[:nrep], seeds, k, mode).tolist() == want.tolist(), (k, mode, nrep)
    assert k_hop_count_multi(reps, seeds[:2], 2).tolist() == k_hop_count_batch(g, seeds[:2], 2).tolist()
    assert k_hop_count_multi(reps, [], 2).tolist() == []
    with pytest.raises(ContractError, match="k-hop seed 99999999 is not an allocated node"):
        k_hop_count_multi(reps, [int(seeds[0]), 99999999], 2)
    with pytest.raises(ContractError, match=r"k-hop count 0 outside \[1, 32\]"):
        k_hop_count_multi(reps, seeds, 0)


@pytest.mark.parametrize("strag", ["0", "2", "32", "4096", "100000000"])
def test_straggler_thresholds(strag):
    """The LANES engine's straggler lanes (lanes with at most m / MGK_STRAG
    frontier out-edges push while the others pull, mgk_ms.cu): off, nearly every
    lane a straggler, the default, and thresholds only tiny frontiers meet --
    all give the oracle's counts, in every narrow lane-word width."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    worker = Path(__file__).resolve().parent / "helpers" / "strag_worker.py"
    env = dict(os.environ, MGK_STRAG=strag)
    r = subprocess.run([sys.executable, str(worker)], stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True,
                       env=env, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:]


def test_two_processes_share_one_gpu():
    """Regression: workspace zeroing ran on the legacy stream, unordered with
    the engines' non-blocking streams; with another process on the GPU the
    first traversal could start on recycled, non-zero bitmaps."""
    import subprocess
    import sys
    from pathlib import Path
    worker = Path(__file__).resolve().parent / "helpers" / "share_worker.py"
    procs = [subprocess.Popen([sys.executable, str(worker)], stdout=subprocess.PIPE, stderr=subprocess.STDOUT,
                              text=True) for _ in range(2)]
    outs = [p.communicate(timeout=600)[0] for p in procs]
    assert all(p.returncode == 0 for p in procs), outs


def test_concurrent_host_calls_on_one_graph(g1):
    """The reference's server runs queries from several worker threads against
    one graph (server.cpp:75-76): calls are reentrant (own workspace and
    stream each) and answer exactly like sequential calls."""
    from concurrent.futures import ThreadPoolExecutor
    rp, ci, g = g1
    jobs = [(H.pick_seeds(rp, 50 + 7 * i, 100 + i), 1 + i % 4, i % 2) for i in range(16)]
    want = [k_hop_count_batch(g, s, k, m).tolist() for s, k, m in jobs]
    with ThreadPoolExecutor(max_workers=8) as ex:
        for _ in range(3):
            got = list(ex.map(lambda j: k_hop_count_batch(g, j[0], j[1], j[2]).tolist(), jobs))
            assert got == want


def test_sections_in_one_call(port, g1):
    """mgk_khop_count_ks: several k for one seed list in one call (SINGLE and
    LANES windows mixed) equals one call per k; errors in the reference order."""
    from paper_1905_01294_b200 import k_hop_count_sections
    rp, ci, g = g1
    seeds = H.pick_seeds(rp, 300, 2)
    for mode in (0, 1):
        ks = [1, 2, 3, 6, 2]
        got = k_hop_count_sections(g, seeds, ks, mode)
        assert got.shape == (len(ks), len(seeds))
        for j, k in enumerate(ks):
            assert got[j].tolist() == k_hop_count_batch(g, seeds, k, mode).tolist(), (mode, k)
    assert k_hop_count_sections(g, seeds[:1], [2], 0)[0].tolist() == oracle_counts(port, rp, ci, seeds[:1], 2, 0)
    with pytest.raises(ContractError, match=r"k-hop count 40 outside \[1, 32\]"):
        k_hop_count_sections(g, seeds, [1, 40], 0)

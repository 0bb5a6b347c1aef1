"""CPU: the bench-scale oracle (oracle/bench_oracle.c) pinned to the reference
and to the product's host generator, and the committed bench goldens
(tests/golden/bench_pins.json, made by make_bench_golden.py from oracle/_ref)
checked for internal consistency and against the product's host generator."""
import hashlib
import json

import numpy as np
import pytest

import oracle
from conftest import GOLDEN
from paper_1905_01294_b200 import harness as H

HAVE_REF = oracle.REF_SO.exists()
PINS = GOLDEN / "bench_pins.json"


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


SPECS = [H.G1, H.GraphSpec("s14u", scale=14, target_unique=150_000, relabel=2, rng_seed=5),
         H.GraphSpec("s13r0", scale=13, relabel=0, rng_seed=9)]


@pytest.mark.parametrize("spec", SPECS, ids=lambda s: s.name)
def test_oracle_generator_matches_product_host_generator(port, spec):
    rp, ci = port.gen_spec(spec)
    rp2, ci2 = H.gen_csr(spec)
    assert np.array_equal(rp, rp2) and np.array_equal(ci, ci2)
    # CSR invariants (sparse.hpp:80-82): strictly ascending columns, no loops
    deg = np.diff(rp.astype(np.int64))
    rows = np.repeat(np.arange(len(deg)), deg)
    assert (ci < len(rp) - 1).all() and not (ci == rows).any()
    same_row = rows[1:] == rows[:-1]
    assert (ci[1:][same_row] > ci[:-1][same_row]).all()
    if spec.target_unique:
        assert len(ci) == spec.target_unique
    if spec.relabel == 2:
        indeg = np.bincount(ci, minlength=len(deg))
        assert ((deg + indeg) > 0).all()  # no isolated vertex survives


def test_pick_seeds_u32_matches_product(port):
    rp, _ = port.gen_spec(SPECS[1])
    for n, rng in ((1, 1), (300, 1), (1000, 7)):
        assert np.array_equal(port.pick_seeds_u32(rp, n, rng), H.pick_seeds(rp, n, rng))
    # prefix stability (bench.hpp:122-125)
    assert np.array_equal(port.pick_seeds_u32(rp, 10, 1), port.pick_seeds_u32(rp, 300, 1)[:10])


@pytest.mark.skipif(not HAVE_REF, reason="reference not built here")
def test_pick_seeds_u32_matches_reference(port):
    R = oracle.Ref()
    rp, ci = port.gen_spec(SPECS[1])
    src, dst = H.csr_to_edges(rp, ci)
    g = R.build_bench_graph(src, dst, len(rp) - 1)
    for n, rng in ((300, 1), (77, 3)):
        assert port.pick_seeds_u32(rp, n, rng).tolist() == g.pick_seeds(n, rng).tolist()


@pytest.mark.skipif(not HAVE_REF, reason="reference not built here")
def test_khop_many_matches_reference_both_routes(port):
    R = oracle.Ref()
    rp, ci = port.gen_spec(SPECS[1])
    seeds = port.pick_seeds_u32(rp, 40, 2)
    src, dst = H.csr_to_edges(rp, ci)
    g = R.build_bench_graph(src, dst, len(rp) - 1)
    M = R.matrix(rp, ci)
    for k in (1, 2, 3, 6, 32):
        ex, cu, E, lv = port.khop_many(rp, ci, seeds, k, threads=3, work=True)
        for mode, got in ((0, ex), (1, cu)):
            want_m, _ = M.khop_jobs(seeds, np.full(len(seeds), k, np.uint32), mode, threads=2)
            want_g, _ = g.khop_jobs(seeds, np.full(len(seeds), k, np.uint32), mode, threads=2)
            assert got.tolist() == want_m.tolist() == want_g.tolist(), (k, mode)
        # level sizes: exact at every k' <= k, cumulative = their sum
        assert (lv[:, 0] == 1).all()
        assert lv[:, 1:].sum(axis=1).tolist() == cu.tolist()
        for s_i, s in enumerate(seeds[:5]):
            e_ref, sizes = port.khop_work(rp.astype(np.uint64), ci.astype(np.uint64), int(s), k)
            assert E[s_i] == e_ref and lv[s_i, :len(sizes)].tolist() == sizes.tolist()


@pytest.mark.skipif(not HAVE_REF, reason="reference not built here")
def test_matrix_route_errors_are_the_references():
    R = oracle.Ref()
    M = R.matrix(np.array([0, 1, 1], np.uint32), np.array([1], np.uint32))
    with pytest.raises(oracle.RefError, match="k-hop seed 2 is not an allocated node"):
        M.khop_jobs([2], [1])
    with pytest.raises(oracle.RefError, match=r"k-hop count 33 outside \[1, 32\]"):
        M.khop_jobs([0], [33])


@pytest.mark.skipif(not PINS.exists(), reason="bench goldens not generated")
def test_bench_pins_consistent():
    p = json.loads(PINS.read_text())
    g2 = p["G2"]
    assert g2["n"] == 2_412_345 and g2["m"] == 67_108_864
    r = g2["ref"]
    assert len(r["cfg2"]["counts"]["1"]["exact"]) == 300 and len(r["cfg3"]["counts"]["6"]["exact"]) == 10
    # cfg3's seeds are the prefix of cfg2's (prefix-stable pick_seeds)
    for k in ("1", "2"):
        c = r["cfg2"]["counts"][k]
        if k == "1":  # k = 1: exact == cumulative
            assert c["exact"] == c["cumulative"]
        assert all(e <= cu for e, cu in zip(c["exact"], c["cumulative"]))
    lv = np.array(g2["cfg5"]["levels"])
    assert lv.shape == (3 * 512, 6)
    # cfg5 sample batch 0 = the first 512 seeds: its first 300 levels agree with cfg2 / cfg3
    assert lv[:300, 0].tolist() == r["cfg2"]["counts"]["1"]["exact"]
    assert lv[:300, 1].tolist() == r["cfg2"]["counts"]["2"]["exact"]
    assert lv[:300, :2].sum(1).tolist() == r["cfg2"]["counts"]["2"]["cumulative"]
    assert lv[:10, 2].tolist() == r["cfg3"]["counts"]["3"]["exact"]
    assert lv[:10, 5].tolist() == r["cfg3"]["counts"]["6"]["exact"]
    assert lv[:10].sum(1).tolist() == r["cfg3"]["counts"]["6"]["cumulative"]
    if "G4" in p:
        g4 = p["G4"]
        assert g4["m"] == 1_470_000_000
        assert len(g4["ref"]["cfg4_k12"]["counts"]["2"]["exact"]) == 300
        assert len(g4["ref"]["cfg4_k36"]["counts"]["6"]["exact"]) == 20


@pytest.mark.skipif(not PINS.exists(), reason="bench goldens not generated")
def test_product_host_generator_matches_pinned_g2(port):
    """The product's host generator (mgk_gen_rmat_csr) builds exactly the G2
    the reference counts were pinned on; seeds likewise."""
    p = json.loads(PINS.read_text())["G2"]
    rp, ci = H.gen_csr(H.G2)
    assert len(rp) - 1 == p["n"] and sha(rp, ci) == p["csr_sha256"]
    master = H.pick_seeds(rp, 65536, 1)
    assert master[:300].tolist() == p["seeds300"] and sha(master) == p["seeds65536_sha256"]

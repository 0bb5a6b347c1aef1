"""GRAPHSNAP1 load: the reference's snapshot grammar
(proj/core/src/snapshot.cpp:162-231) pinned by tests/golden/snapshot_pins.json,
which make_golden.py produced with the reference's own parser and writer.

CPU tests run the host-side grammar inside libmgk.so (mgk_snapshot_check) and
the bench-graph writer; the gpu tests load the same texts through the GPU
parser (mgk_graph_load_snapshot) and compare matrices, counts and messages."""
import hashlib

import numpy as np
import pytest

from conftest import load_golden
from paper_1905_01294_b200 import SnapshotError, harness as H, snapshot_check


@pytest.fixture(scope="module")
def pins():
    return load_golden("snapshot_pins")


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def edges_declared(text: bytes) -> int:
    lines = text.split(b"\n")
    n = int(lines[1][6:])
    return int(lines[2 + n][6:])


def test_host_grammar_valid(pins):
    for case in pins["valid"]:
        t = case["text"].encode()
        assert snapshot_check(t) == (case["node_count"], edges_declared(t)), case["name"]


def test_host_grammar_errors(pins):
    for case in pins["errors"]:
        with pytest.raises(SnapshotError) as ex:
            snapshot_check(case["text"].encode())
        assert str(ex.value) == case["error"], case["name"]


def test_bench_writer_is_the_reference_writer(port, pins):
    b = pins["bench"]
    src, dst = port.rmat_generate(b["scale"], rng_seed=b["rng_seed"])
    n = 1 << b["scale"]
    rp, ci = port.build_csr(n, src, dst)
    text = H.snapshot_text(rp, ci, n)
    assert len(text) == b["bytes"]
    assert hashlib.sha256(text).hexdigest() == b["text_sha256"]
    assert snapshot_check(text) == (n, len(ci))


# ---- the GPU loader ----------------------------------------------------------------------
@pytest.mark.gpu
def test_gpu_load_valid(pins):
    from paper_1905_01294_b200 import DeviceGraph
    for case in pins["valid"]:
        t = case["text"].encode()
        for rel, want in case["csr"].items():
            g = DeviceGraph.from_snapshot(t, relation=None if rel == "ANY" else rel)
            assert g.node_count == case["node_count"]
            rp, ci = g.csr()
            assert rp.tolist() == want["row_ptr"], (case["name"], rel)
            assert ci.tolist() == want["col_idx"], (case["name"], rel)


@pytest.mark.gpu
def test_gpu_load_errors(pins, tmp_path):
    from paper_1905_01294_b200 import DeviceGraph
    for case in pins["errors"]:
        with pytest.raises(SnapshotError) as ex:
            DeviceGraph.from_snapshot(case["text"].encode())
        assert str(ex.value) == case["error"], case["name"]
    missing = tmp_path / "nope.snap"
    with pytest.raises(SnapshotError, match=f"cannot open '{missing}' for reading"):
        DeviceGraph.from_snapshot(path=missing)


@pytest.mark.gpu
def test_gpu_load_bench_graph(port, pins, tmp_path):
    from paper_1905_01294_b200 import DeviceGraph, k_hop_count_batch
    b = pins["bench"]
    src, dst = port.rmat_generate(b["scale"], rng_seed=b["rng_seed"])
    n = 1 << b["scale"]
    rp, ci = port.build_csr(n, src, dst)
    f = tmp_path / "bench.snap"
    f.write_bytes(H.snapshot_text(rp, ci, n))
    for rel, key in ((None, "any_csr_sha256"), ("EDGE", "edge_csr_sha256")):
        g = DeviceGraph.from_snapshot(path=f, relation=rel)
        drp, dci = g.csr()
        assert sha(drp.astype(np.uint64), dci.astype(np.uint64)) == b[key]
    assert k_hop_count_batch(g, b["seeds"], 2).tolist() == b["counts_k2"]


@pytest.mark.gpu
def test_gpu_load_round_trip_g1():
    """Size-independent property at a bigger size: CSR -> text -> GPU parse ->
    the same CSR, for ANY and the relation, and an unknown relation is empty."""
    from paper_1905_01294_b200 import DeviceGraph
    rp, ci = H.gen_csr(H.G1)
    text = H.snapshot_text(rp, ci, relation="EDGE")
    for rel in (None, "EDGE"):
        g = DeviceGraph.from_snapshot(text, relation=rel)
        drp, dci = g.csr()
        assert np.array_equal(drp, rp) and np.array_equal(dci, ci)
    g = DeviceGraph.from_snapshot(text, relation="OTHER")
    drp, dci = g.csr()
    assert int(drp[-1]) == 0 and len(drp) == len(rp)
    # one malformed line deep in the edge section is found and named
    lines = text.split(b"\n")
    k = len(lines) - 1000
    bad = b"\n".join(lines[:k] + [lines[k].replace(b"EDGE", b"ED-GE")] + lines[k + 1:])
    with pytest.raises(SnapshotError) as ex:
        DeviceGraph.from_snapshot(bad)
    assert str(ex.value) == f"snapshot parse error at line {k + 1}: relation type 'ED-GE' is not a valid identifier"

"""The C-ABI library loads and exports every symbol include/mgk.h declares
(no compute calls: this runs without a GPU), and the host-side helpers."""
import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

from paper_1905_01294_b200 import _lib, harness as H
from paper_1905_01294_b200.khop import ContractError, HarnessError

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "mgk.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mgk_\w+)\s*\(", text)))


def test_header_symbols_exported():
    L = _lib.lib()
    names = declared_symbols()
    assert len(names) >= 18
    for name in names:
        assert hasattr(L, name), name
    bound = {n for n, _, _ in _lib.SIGNATURES}
    assert set(names) == bound, set(names) ^ bound


def test_abi_version_and_no_gpu_is_loud():
    L = _lib.lib()
    assert L.mgk_abi_version() == 2
    if L.mgk_device_count() == 0:
        h = C.c_void_p()
        rp = np.array([0, 0], np.uint32)
        rc = L.mgk_graph_upload_u32(0, 1, 0, rp.ctypes.data, rp.ctypes.data, C.byref(h))
        assert rc == _lib.MGK_ECUDA
        assert "no CUDA device" in _lib.last_error()


def test_device_sections_validation_before_device_work():
    """mgk_khop_count_device_ks checks its arguments before touching the graph."""
    L = _lib.lib()
    ks = np.array([1, 2], np.uint32)
    assert L.mgk_khop_count_device_ks(None, None, 0, ks.ctypes.data, 2, 0, None, None) == _lib.MGK_ECONTRACT
    assert "null graph" in _lib.last_error()
    fake = C.c_void_p(8)  # never dereferenced: every case below fails first
    assert L.mgk_khop_count_device_ks(fake, None, 0, None, 2, 0, None, None) == _lib.MGK_ECONTRACT
    assert "null argument" in _lib.last_error()
    assert L.mgk_khop_count_device_ks(fake, None, 0, ks.ctypes.data, 2, 7, None, None) == _lib.MGK_ECONTRACT
    assert "unknown traverse mode 7" in _lib.last_error()
    for bad in (0, 33):
        kb = np.array([1, bad], np.uint32)
        assert L.mgk_khop_count_device_ks(fake, None, 0, kb.ctypes.data, 2, 0, None, None) == _lib.MGK_ECONTRACT
        assert f"k-hop count {bad} outside [1, 32]" in _lib.last_error()


def test_upload_validation_messages():
    L = _lib.lib()
    h = C.c_void_p()
    rp = np.array([0, 2, 1], np.uint64)
    ci = np.array([1, 0], np.uint64)
    assert L.mgk_graph_upload(0, 2, 2, rp.ctypes.data, ci.ctypes.data, C.byref(h)) == _lib.MGK_ECONTRACT
    assert "row_ptr must start at 0 and end at nnz" in _lib.last_error()
    rp = np.array([0, 1, 2], np.uint64)
    ci = np.array([1, 5], np.uint64)
    assert L.mgk_graph_upload(0, 2, 2, rp.ctypes.data, ci.ctypes.data, C.byref(h)) == _lib.MGK_ECONTRACT
    assert "column 5 out of range for 2 rows" in _lib.last_error()


def test_pick_seeds_matches_oracle(port, pins):
    for p in pins["pick_seeds"]:
        src, dst = port.rmat_generate(p["scale"], rng_seed=p["rng_seed"])
        rp, _ = port.build_csr(1 << p["scale"], src, dst)
        assert H.pick_seeds(rp.astype(np.uint32), p["n"], p["seed_rng"]).tolist() == p["seeds"]
    rp = np.array([0, 1, 1, 1], np.uint32)
    with pytest.raises(HarnessError, match="need 2 seeds but only 1 nodes have out-degree >= 1"):
        H.pick_seeds(rp, 2, 1)


def test_generator_deterministic_and_clean():
    spec = H.GraphSpec("t", scale=12, edge_factor=8, target_unique=20000, relabel=2, rng_seed=5)
    rp, ci = H.gen_csr(spec)
    rp2, ci2 = H.gen_csr(spec)
    assert (rp == rp2).all() and (ci == ci2).all()
    assert len(ci) == 20000
    src, dst = H.csr_to_edges(rp, ci)
    assert (src != dst).all()
    keys = src.astype(np.uint64) << 32 | dst
    assert (np.diff(keys.astype(np.int64)) > 0).all()  # sorted, no duplicates
    n = len(rp) - 1
    touched = np.zeros(n, bool)
    touched[src] = True
    touched[dst] = True
    assert touched.all()  # relabel=2 leaves no isolated ids
    other = H.gen_csr(H.GraphSpec("t", scale=12, edge_factor=8, target_unique=20000, relabel=2, rng_seed=6))
    assert len(other[1]) != len(ci) or not np.array_equal(other[1], ci)


def test_generator_raw_mode_counts():
    spec = H.GraphSpec("t", scale=10, edge_factor=4, target_unique=0, relabel=1)
    rp, ci = H.gen_csr(spec)
    assert len(rp) - 1 == 1024
    assert 0 < len(ci) <= 4096


def test_mxm_validation_before_device_work(tmp_path):
    """mgk_mxm checks shapes with the reference's messages (sparse.cpp:294-301)
    before touching a device, so these run without a GPU."""
    from conftest import load_golden
    from paper_1905_01294_b200 import mxm
    for e in load_golden("mxm_pins")["errors"]:
        a, b, m = e["a"], e["b"], e["mask"]
        A = (a[0], a[1], np.zeros(a[0] + 1, np.uint64), np.zeros(0, np.uint64), None)
        B = (b[0], b[1], np.zeros(b[0] + 1, np.uint64), np.zeros(0, np.uint64), None)
        M = None if m is None else (m[0], m[1], np.zeros(m[0] + 1, np.uint64), np.zeros(0, np.uint64), None)
        with pytest.raises(ContractError) as ex:
            mxm(A, B, 0, M)
        assert str(ex.value) == e["error"]
    A = (2, 2, np.array([0, 1, 1], np.uint64), np.array([5], np.uint64), None)
    with pytest.raises(ContractError, match="mxm: A column out of range"):
        mxm(A, A)
    with pytest.raises(ContractError, match="unknown semiring 7"):
        mxm(A, A, 7)


def test_snapshot_writer_and_checker_round_trip():
    """Host-only: the bench-graph writer's text passes the exact grammar and
    reports its own node / edge counts."""
    from paper_1905_01294_b200 import snapshot_check
    rp, ci = H.gen_csr(H.GraphSpec("S10", scale=10, edge_factor=8, relabel=1))
    text = H.snapshot_text(rp, ci, relation="KNOWS")
    assert snapshot_check(text) == (len(rp) - 1, len(ci))
    assert text.startswith(b"GRAPHSNAP1\nNODES ")

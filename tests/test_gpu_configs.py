"""GPU parity on every BASELINE.json bench config at FULL size, bit for bit
against the reference's own counts (tests/golden/bench_pins.json, made from
oracle/_ref by make_bench_golden.py; acceptance_main.cpp:53-88 style).

* the bench graphs are generated ON THE GPU (mgk_graph_gen_rmat, the path
  bench.py uses) and their CSR must hash equal to the oracle generator's
  (an independent C restatement) — a generator bug cannot hide;
* cfg2: all 300 seeds x k=1,2, exact + cumulative, through the host API, the
  host sections call and the device-resident sections call bench.py times;
* cfg3: all 10 seeds x k=3,6, both modes, both engines;
* cfg4: G4 (1.47B edges) — 300 seeds x k=1,2 and 20 seeds x k=3,6, both
  modes, through the schedule call bench.py times;
* cfg5: the 65,536-seed list in W=8 lane batches (512 seeds each), k=2,3,6
  exact and k=6 cumulative; the 1,536 seeds of batches 0, 64 and 127 are
  compared with the oracle's per-level sizes.
"""
import hashlib
import json

import numpy as np
import pytest

from conftest import GOLDEN
from paper_1905_01294_b200 import (ENGINE_LANES, ENGINE_SINGLE, DeviceGraph, Tuning, device_check, harness as H,
                                   k_hop_count_batch, k_hop_count_device, k_hop_count_device_schedule,
                                   k_hop_count_device_sections, k_hop_count_schedule, k_hop_count_sections)

pytestmark = pytest.mark.gpu
PINS = json.loads((GOLDEN / "bench_pins.json").read_text()) if (GOLDEN / "bench_pins.json").exists() else {}
need = pytest.mark.skipif(not PINS, reason="tests/golden/bench_pins.json missing")


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def ref(graph, label, k, mode):
    return PINS[graph]["ref"][label]["counts"][str(k)][("exact", "cumulative")[mode]]


@pytest.fixture(scope="module")
def g2():
    g = DeviceGraph.generate(H.G2)
    rp, ci = g.csr()
    return rp, ci, g


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    return torch


@need
def test_g2_generated_on_gpu_is_the_pinned_graph(g2):
    rp, ci, g = g2
    p = PINS["G2"]
    assert g.nrows == p["n"] and g.nnz == p["m"]
    assert sha(rp, ci) == p["csr_sha256"]
    assert H.pick_seeds(rp, 300, 1).tolist() == p["seeds300"]


@need
@pytest.mark.parametrize("mode", [0, 1])
def test_cfg2_all_seeds(g2, torch_cuda, mode):
    torch = torch_cuda
    _, _, g = g2
    seeds = np.array(PINS["G2"]["seeds300"], np.uint64)
    want = {k: ref("G2", "cfg2", k, mode) for k in (1, 2)}
    for k in (1, 2):
        assert k_hop_count_batch(g, seeds, k, mode).tolist() == want[k], k
        assert k_hop_count_batch(g, seeds, k, mode, engine=ENGINE_SINGLE).tolist() == want[k], k
    sec = k_hop_count_sections(g, seeds, [1, 2], mode)
    assert [s.tolist() for s in sec] == [want[1], want[2]]
    # the device-resident sections call bench.py times (k = 1 rides on the k = 2 launch)
    d_seeds = torch.from_numpy(seeds.astype(np.int32)).cuda()
    d_out = torch.zeros(600, dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream()
    k_hop_count_device_sections(g, d_seeds.data_ptr(), 300, [1, 2], mode, d_out.data_ptr(), st.cuda_stream)
    device_check(g, st.cuda_stream)
    out = d_out.cpu().numpy()
    assert out[:300].tolist() == want[1] and out[300:].tolist() == want[2]


@need
@pytest.mark.parametrize("mode", [0, 1])
def test_cfg3_all_seeds(g2, mode):
    _, _, g = g2
    seeds = np.array(PINS["G2"]["seeds300"][:10], np.uint64)
    for k in (3, 6):
        want = ref("G2", "cfg3", k, mode)
        assert k_hop_count_batch(g, seeds, k, mode).tolist() == want, k
        assert k_hop_count_batch(g, seeds, k, mode, engine=ENGINE_LANES).tolist() == want, k
        assert k_hop_count_batch(g, seeds, k, mode, engine=ENGINE_SINGLE).tolist() == want, k
    # both sections from one shared traversal (the schedule call)
    got = k_hop_count_schedule(g, seeds, [10, 10], [3, 6], mode)
    assert [x.tolist() for x in got] == [ref("G2", "cfg3", 3, mode), ref("G2", "cfg3", 6, mode)]


@need
@pytest.mark.parametrize("W", [8, 0])
def test_cfg5_sampled_batches(g2, torch_cuda, W):
    """65,536 seeds in lane batches (W=8: 512 seeds per batch; W=0: auto), all
    seeds run, the 1,536 seeds of batches 0, 64, 127 checked."""
    torch = torch_cuda
    rp, _, g = g2
    p = PINS["G2"]
    master = H.pick_seeds(rp, 65536, 1)
    assert sha(master) == p["seeds65536_sha256"]
    lv = np.array(p["cfg5"]["levels"], np.uint64)  # [1536, 6] = |F_1..F_6|
    B = p["cfg5"]["batch_seeds"]
    idx = np.concatenate([np.arange(b * B, (b + 1) * B) for b in p["cfg5"]["batches"]])
    d_seeds = torch.from_numpy(master.astype(np.int32)).cuda()
    d_counts = torch.zeros(len(master), dtype=torch.int64, device="cuda")
    sp = torch.cuda.current_stream().cuda_stream
    try:
        g.set_tuning(Tuning(lanes_words=W))
        for k, mode, want in ((2, 0, lv[:, 1]), (3, 0, lv[:, 2]), (6, 0, lv[:, 5]), (6, 1, lv.sum(1))):
            k_hop_count_device(g, d_seeds.data_ptr(), len(master), k, mode, d_counts.data_ptr(), sp)
            device_check(g, sp)
            got = d_counts.cpu().numpy().astype(np.uint64)[idx]
            assert np.array_equal(got, want), (k, mode, int(np.flatnonzero(got != want)[0]))
    finally:
        g.set_tuning(Tuning())


@need
def test_schedule_equals_per_k_calls(g2, torch_cuda):
    """mgk_khop_count_schedule (sections over prefixes of one master list,
    bench.cpp:311-343) == one batch call per section, host and device."""
    torch = torch_cuda
    rp, _, g = g2
    seeds = H.pick_seeds(rp, 300, 1)
    ns, ks = [300, 300, 10, 10], [1, 2, 3, 6]
    got = k_hop_count_schedule(g, seeds, ns, ks, 0)
    for n, k, x in zip(ns, ks, got):
        assert x.tolist() == k_hop_count_batch(g, seeds[:n], k, 0).tolist(), k
    d_seeds = torch.from_numpy(seeds.astype(np.int32)).cuda()
    d_out = torch.zeros(sum(ns), dtype=torch.int64, device="cuda")
    sp = torch.cuda.current_stream().cuda_stream
    k_hop_count_device_schedule(g, d_seeds.data_ptr(), ns, ks, 0, d_out.data_ptr(), sp)
    device_check(g, sp)
    assert d_out.cpu().numpy().astype(np.uint64).tolist() == np.concatenate(got).tolist()


# ---- cfg4: the Twitter-shaped G4 (1.47B edges, ~12 GB CSR + CSC) ----------------------------
@pytest.fixture(scope="module")
def g4():
    if "G4" not in PINS:
        pytest.skip("G4 pins not generated")
    g = DeviceGraph.generate(H.G4)
    rp, ci = g.csr()
    yield rp, ci, g
    g.close()


@need
def test_g4_generated_on_gpu_is_the_pinned_graph(g4):
    rp, ci, g = g4
    p = PINS["G4"]
    assert g.nrows == p["n"] and g.nnz == p["m"]
    assert sha(rp, ci) == p["csr_sha256"]
    assert H.pick_seeds(rp, 300, 1).tolist() == p["seeds300"]


@need
@pytest.mark.parametrize("mode", [0, 1])
def test_cfg4_schedule(g4, torch_cuda, mode):
    torch = torch_cuda
    _, _, g = g4
    seeds = np.array(PINS["G4"]["seeds300"], np.uint64)
    ns, ks = [300, 300, 20, 20], [1, 2, 3, 6]
    want = [ref("G4", "cfg4_k12", 1, mode), ref("G4", "cfg4_k12", 2, mode),
            ref("G4", "cfg4_k36", 3, mode), ref("G4", "cfg4_k36", 6, mode)]
    got = k_hop_count_schedule(g, seeds, ns, ks, mode)
    assert [x.tolist() for x in got] == want
    d_seeds = torch.from_numpy(seeds.astype(np.int32)).cuda()
    d_out = torch.zeros(sum(ns), dtype=torch.int64, device="cuda")
    sp = torch.cuda.current_stream().cuda_stream
    k_hop_count_device_schedule(g, d_seeds.data_ptr(), ns, ks, mode, d_out.data_ptr(), sp)
    device_check(g, sp)
    assert d_out.cpu().numpy().astype(np.uint64).tolist() == sum(want, [])


@need
def test_cfg4_single_engine_deep(g4):
    """The per-seed engine on G4 at depth agrees with the reference too."""
    _, _, g = g4
    seeds = np.array(PINS["G4"]["seeds300"][:3], np.uint64)
    for k in (3, 6):
        assert k_hop_count_batch(g, seeds, k, 0, engine=ENGINE_SINGLE).tolist() == \
            ref("G4", "cfg4_k36", k, 0)[:3], k

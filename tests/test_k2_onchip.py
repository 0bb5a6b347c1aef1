"""The k = 2 on-chip path (mgk_k2.cu: per-seed visited sets in shared memory)
against the oracle, including the cases it handles specially: seeds cut over
several CTA groups (hubs), a work line shorter than the group count, the F1
scratch running out, isolated seeds and self loops."""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from paper_1905_01294_b200 import ENGINE_SINGLE, DeviceGraph, Tuning, harness as H, k_hop_count_batch

pytestmark = pytest.mark.gpu
WORKER = Path(__file__).resolve().parent / "helpers" / "k2_worker.py"


@pytest.mark.parametrize("env", [
    {},                                                # defaults
    {"MGK_K2_SEEDCOST": "0"},                          # pure entry split: many cut seeds
    {"MGK_K2_SEEDCOST": "0", "MGK_K2_F1CAP": "64"},    # F1 scratch runs out: in-kernel prefixes
    {"MGK_K2_SEEDCOST": "100000000"},                  # one seed per group at most
    {"MGK_K2_SNAP": "1"},                              # boundaries snap to seed edges a whole group away
    {"MGK_K2_SNAP": "1000000", "MGK_K2_SEEDCOST": "0"},  # (almost) no snapping
    {"MGK_K2_SLICE_WORDS": "256"},                     # G1 in 8 slices (the split array path, R > 2)
    {"MGK_K2_SLICE_WORDS": "1024", "MGK_K2_SEEDCOST": "0"},  # G1 in 2 slices
    {"MGK_NO_K2SMEM": "1"},                            # the L2-bitmap engine (fr_kernel)
], ids=["default", "cost0", "f1cap", "cost_huge", "snap_wide", "snap_none", "r8", "r2",
                      "no_onchip"])
def test_k2_paths_against_oracle(env):
    p = subprocess.run([sys.executable, str(WORKER)], env={**os.environ, **env}, capture_output=True,
                       text=True, timeout=900)
    assert p.returncode == 0, p.stdout + p.stderr


def test_k2_stats_and_agreement(port):
    rp, ci = H.gen_csr(H.G1)
    g = DeviceGraph.from_csr(rp, ci)
    seeds = H.pick_seeds(rp, 2000, 3)  # several seeds per group
    counts, st = k_hop_count_batch(g, seeds, 2, 0, stats=True)
    assert st["launches"] == 1 and st["path"] == "smem_k2"
    assert st["levels"][2]["frontier"] == int(counts.sum())
    rp64, ci64 = rp.astype(np.uint64), ci.astype(np.uint64)
    e = sum(port.khop_work(rp64, ci64, int(s), 2)[0] for s in seeds)
    assert st["levels"][1]["edges"] + st["levels"][2]["edges"] == e
    # forced directions run the general engine: same answers
    for d in (1, 2):
        g.set_tuning(Tuning(force_dir=d))
        assert k_hop_count_batch(g, seeds, 2, 0, engine=ENGINE_SINGLE).tolist() == counts.tolist()
    g.set_tuning(Tuning())
    cum = k_hop_count_batch(g, seeds, 2, 1)
    one = k_hop_count_batch(g, seeds, 1, 0)
    assert (cum == counts + one).all()


def test_sections_share_the_k2_launch():
    """k = 1 sections answered by the on-chip k = 2 launch (|F1| is part of it):
    host and device sections agree with separate per-k calls, in any order,
    with and without other sections, and when the fusion does not apply."""
    import torch
    from paper_1905_01294_b200 import k_hop_count_device_sections, k_hop_count_sections
    rp, ci = H.gen_csr(H.G1)
    g = DeviceGraph.from_csr(rp, ci)
    seeds = H.pick_seeds(rp, 700, 4)
    for mode in (0, 1):
        ref = {k: k_hop_count_batch(g, seeds, k, mode, engine=ENGINE_SINGLE if k < 3 else 0) for k in (1, 2, 3)}
        for ks in ([1, 2], [2, 1], [1, 2, 3], [3, 1, 2], [1], [2], [1, 1, 2]):
            got = k_hop_count_sections(g, seeds, ks, mode)
            assert all((got[j] == ref[k]).all() for j, k in enumerate(ks)), (mode, ks)
            d_seeds = torch.from_numpy(seeds.astype(np.int32)).cuda()
            d_counts = torch.zeros(len(ks) * len(seeds), dtype=torch.int64, device="cuda")
            k_hop_count_device_sections(g, d_seeds.data_ptr(), len(seeds), ks, mode, d_counts.data_ptr(),
                                        torch.cuda.current_stream().cuda_stream)
            torch.cuda.synchronize()
            dc = d_counts.cpu().numpy().astype(np.uint64).reshape(len(ks), len(seeds))
            assert all((dc[j] == ref[k]).all() for j, k in enumerate(ks)), ("device", mode, ks)
    g.set_tuning(Tuning(force_dir=1))  # general engine for k = 2: no fusion, same answers
    got = k_hop_count_sections(g, seeds, [1, 2], 0)
    assert (got[0] == k_hop_count_batch(g, seeds, 1, 0)).all() and (got[1] == k_hop_count_batch(g, seeds, 2, 0)).all()

"""Child process for tests/test_k2_onchip.py: k = 2 counts under the
environment the parent set (MGK_K2_SEEDCOST, MGK_K2_F1CAP, MGK_NO_K2SMEM are
read once per process), checked against the C oracle. Exit 0 = all equal."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import oracle  # noqa: E402  (the checker)
from paper_1905_01294_b200 import DeviceGraph, harness as H, k_hop_count_batch, walk_count_batch  # noqa: E402

port = oracle.Port()
bad = 0


def check(rp, ci, seeds, label):
    global bad
    g = DeviceGraph.from_csr(rp, ci)
    rp64, ci64 = rp.astype(np.uint64), ci.astype(np.uint64)
    for mode in (0, 1):
        want = [port.khop_count(rp64, ci64, int(s), 2, mode) for s in seeds]
        got = k_hop_count_batch(g, seeds, 2, mode).tolist()
        if got != want:
            bad += 1
            print(label, "mode", mode, "mismatch at", [i for i, (a, b) in enumerate(zip(got, want)) if a != b][:10])
    for lo in (1, 2):  # walk_targets windows [1, 2] and [2, 2]: nothing pre-visited
        want = [len(port.walk_targets(rp64, ci64, int(s), lo, 2)) for s in seeds]
        got = walk_count_batch(g, seeds, lo, 2).tolist()
        if got != want:
            bad += 1
            print(label, "walk", lo, "mismatch at", [i for i, (a, b) in enumerate(zip(got, want)) if a != b][:10])


rp, ci = H.gen_csr(H.G1)
deg = np.diff(rp)
check(rp, ci, H.pick_seeds(rp, 300, 1), "cfg1")
hubs = np.argsort(deg)[-40:]  # heavy seeds: cut over many groups
check(rp, ci, np.concatenate([hubs, H.pick_seeds(rp, 60, 5), hubs[:5]]), "hubs")
check(rp, ci, np.array([int(hubs[-1])]), "one hub")
iso = np.flatnonzero(deg == 0)[:4]
check(rp, ci, np.concatenate([iso, H.pick_seeds(rp, 3, 9), iso]), "isolated")
# self loops and a tiny graph (work line shorter than the group count)
loops_rp = np.array([0, 2, 4, 5, 6], np.uint32)
loops_ci = np.array([0, 1, 1, 2, 3, 0], np.uint32)
check(loops_rp, loops_ci, np.array([0, 1, 2, 3, 0]), "loops")
print("mismatching checks", bad)
sys.exit(1 if bad else 0)

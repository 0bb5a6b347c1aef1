"""Child process for test_straggler_thresholds: LANES counts (one word per
vertex: 8 / 10 / 16 / 64-bit lane words) under the MGK_STRAG threshold given in
the environment, against the CPU oracle. MGK_STRAG is read once per process,
hence the child. Exit code 0 = every count equals the oracle's."""
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import oracle  # noqa: E402  (the checker)
from paper_1905_01294_b200 import ENGINE_LANES, DeviceGraph, harness as H, k_hop_count_batch  # noqa: E402

port = oracle.Port()
rp, ci = H.gen_csr(H.G1)
g = DeviceGraph.from_csr(rp, ci)
rp64, ci64 = rp.astype(np.uint64), ci.astype(np.uint64)
seeds = H.pick_seeds(rp, 64, 5)
deg = np.diff(rp64.astype(np.int64))
# batches mixing hub seeds and low-degree seeds (the stragglers), of every narrow width
order = np.argsort(deg[seeds.astype(np.int64)])
mixed = seeds[np.concatenate([order[:6], order[-6:]])]
groups = [mixed[:10], mixed[1:9], mixed[:12], seeds[:33], seeds[:64]]
bad = 0
for grp in groups:
    for k in (3, 4, 6):
        for mode in (0, 1):
            want = [port.khop_count(rp64, ci64, int(s), k, mode) for s in grp]
            got = k_hop_count_batch(g, grp, k, mode, engine=ENGINE_LANES).tolist()
            if got != want:
                bad += 1
                print("mismatch", os.environ.get("MGK_STRAG"), len(grp), k, mode, got[:4], want[:4])
print("MGK_STRAG", os.environ.get("MGK_STRAG"), "mismatches", bad)
sys.exit(1 if bad else 0)

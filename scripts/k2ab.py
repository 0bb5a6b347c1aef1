"""A/B of on-chip k=2 builds (MGK_LIB_PATH): min/median call time over 12 calls of the
cfg2 (G2) and cfg4 (G4) 300-seed k=2 batches plus a hash of the counts (equal across
builds = same answers). usage: k2ab.py G2 G4"""
import hashlib
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1905_01294_b200 import DeviceGraph, harness as H, k_hop_count_batch  # noqa: E402

for name in sys.argv[1:]:
    g = DeviceGraph.generate(H.SPECS[name])
    rp, _ = g.csr()
    seeds = H.pick_seeds(rp, 300, 1)
    ts = []
    for _ in range(12):
        c, st = k_hop_count_batch(g, seeds, 2, 0, stats=True)
        ts.append(st["kernel_ms"] * 1e3)
    ts = sorted(ts[2:])
    print("%s k2 300 seeds: min %.1f us median %.1f us path %s sha %s" % (
        name, ts[0], ts[len(ts) // 2], st.get("path"), hashlib.sha256(c.tobytes()).hexdigest()[:16]), flush=True)
    del g

"""Timing breakdown of the on-chip k=2 call (G2 = cfg2 by default, or G4): kernel
us, setup (phases 0-1), slices (phase 2), slices + merge, answers; min over 10
calls. usage: k2probe.py [nseeds] [G2|G4]"""
import os
import sys
from pathlib import Path

os.environ.setdefault("MGK_K2_DIAG", "1")  # phase timings in level 0 of the stats

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1905_01294_b200 import DeviceGraph, harness as H, k_hop_count_batch  # noqa: E402

g = DeviceGraph.generate(H.SPECS[sys.argv[2] if len(sys.argv) > 2 else "G2"])
rp, _ = g.csr()
seeds = H.pick_seeds(rp, int(sys.argv[1]) if len(sys.argv) > 1 else 300, 1)
rows = []
for _ in range(12):
    c, st = k_hop_count_batch(g, seeds, 2, 0, stats=True)
    L = st["levels"]
    rows.append((st["kernel_ms"] * 1e3, L[0]["ns"] / 1e3, L[0]["candidates"] / 1e3, L[2]["ns"] / 1e3,
                 st["cleanup_us"], L[0]["frontier"] / 1e3, L[0]["vertices"] / 1e3))
rows = rows[2:]
best = min(rows)
print("k2 call us %.1f | setup %.1f | slices %.1f | slices+merge %.1f | answers %.1f | (0a+bar %.1f 0b+bar %.1f)"
      "  (median call %.1f)" % (*best, sorted(r[0] for r in rows)[len(rows) // 2]))

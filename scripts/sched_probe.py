"""LANES group of the cfg4 schedule (the first 10 of the 300 bench seeds, sections k = 3, 6 in one
traversal) vs the same seeds' exact k = 6 call: device ms and per-hop split (MGK_MS_DIAG=1).
usage: sched_probe.py [G2|G4]"""
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1905_01294_b200 import (DeviceGraph, device_stats, harness as H, k_hop_count_device,  # noqa: E402
                                   k_hop_count_device_schedule)

gname = sys.argv[1] if len(sys.argv) > 1 else "G4"
g = DeviceGraph.generate(H.SPECS[gname])
rp, _ = g.csr()
seeds = torch.from_numpy(H.pick_seeds(rp, 300, 1).astype(np.int32)[:10].copy()).cuda()
out = torch.zeros(20, dtype=torch.int64, device="cuda")
s = torch.cuda.current_stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
calls = {"sections k=3,6": lambda: k_hop_count_device_schedule(g, seeds.data_ptr(), [10, 10], [3, 6], 0, out.data_ptr(), s.cuda_stream),
         "exact k=6": lambda: k_hop_count_device(g, seeds.data_ptr(), 10, 6, 0, out.data_ptr(), s.cuda_stream)}
for name, f in calls.items():
    f()
    ts = []
    for _ in range(5):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        f()
        e1.record(s)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    st = device_stats(g, s.cuda_stream)
    hops = [(h, L["scanned"], round(L["ns"] / 1e3, 1), round(L["union_edges"] / 1e3, 1), round(L["candidates"] / 1e3, 1),
             round(L["edges"] / 1e3, 1)) for h, L in enumerate(st["levels"]) if h and L["runs"]]
    print(f"{gname} {name}: {np.median(ts):.3f} ms {hops}", flush=True)

"""The 10-seed deep group (cfg3 on G2, cfg4 on G4): SINGLE vs LANES at k=3 and
k=6, plus LANES answering both from one traversal; CUDA events, median of 5."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1905_01294_b200 import (ENGINE_LANES, ENGINE_SINGLE, DeviceGraph, device_stats, harness as H,  # noqa: E402
                                   k_hop_count_device)

ns = int(sys.argv[1]) if len(sys.argv) > 1 else 10
for gname in sys.argv[2:] or ["G2", "G4"]:
    g = DeviceGraph.generate(H.SPECS[gname])
    rp, _ = g.csr()
    seeds = H.pick_seeds(rp, ns, 1)
    s = torch.cuda.current_stream()
    d_s = torch.from_numpy(seeds.astype(np.int32)).cuda()
    d_c = torch.zeros(ns, dtype=torch.int64, device="cuda")
    for k in (3, 6):
        for name, eng in (("single", ENGINE_SINGLE), ("lanes", ENGINE_LANES)):
            k_hop_count_device(g, d_s.data_ptr(), ns, k, 0, d_c.data_ptr(), s.cuda_stream, eng)
            ts = []
            for _ in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                k_hop_count_device(g, d_s.data_ptr(), ns, k, 0, d_c.data_ptr(), s.cuda_stream, eng)
                e1.record(s)
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            st = device_stats(g, s.cuda_stream)
            hops = [(h, "pull" if L["pull_runs"] else "push", L["pull_runs"], L["runs"], L["scanned"], round(L["ns"] / 1e3))
                    for h, L in enumerate(st["levels"]) if h and L["runs"]]
            print(f"{gname} {ns} seeds k={k} {name}: {np.median(ts):.3f} ms sum={int(d_c.sum())} {hops}", flush=True)
    del g
    torch.cuda.empty_cache()

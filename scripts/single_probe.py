"""Single-seed deep queries (the reference harness's per-query loop): k=3 and k=6
on G2 / G4 through both engines, CUDA events, median over 5 seeds x 3 reps."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1905_01294_b200 import (ENGINE_LANES, ENGINE_SINGLE, DeviceGraph, harness as H,  # noqa: E402
                                   k_hop_count_device)

for gname in sys.argv[1:] or ["G2", "G4"]:
    g = DeviceGraph.generate(H.SPECS[gname])
    rp, _ = g.csr()
    seeds = H.pick_seeds(rp, 5, 1)
    s = torch.cuda.current_stream()
    d_c = torch.zeros(1, dtype=torch.int64, device="cuda")
    for k in (3, 6):
        for name, eng in (("single", ENGINE_SINGLE), ("lanes", ENGINE_LANES)):
            ts, ans = [], []
            for sd in seeds:
                d_s = torch.tensor([int(sd)], dtype=torch.int32, device="cuda")
                k_hop_count_device(g, d_s.data_ptr(), 1, k, 0, d_c.data_ptr(), s.cuda_stream, eng)
                for _ in range(3):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(s)
                    k_hop_count_device(g, d_s.data_ptr(), 1, k, 0, d_c.data_ptr(), s.cuda_stream, eng)
                    e1.record(s)
                    torch.cuda.synchronize()
                    ts.append(e0.elapsed_time(e1))
                ans.append(int(d_c[0]))
            print(f"{gname} k={k} {name}: median {np.median(ts):.3f} ms answers {ans}", flush=True)
    del g
    torch.cuda.empty_cache()

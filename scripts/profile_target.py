#!/usr/bin/env python3
"""One device-path k-hop launch on G2 for ncu (after two warm-up launches).

usage: profile_target.py [k] [nseeds] [engine: auto|single|lanes] [lanes_words]"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1905_01294_b200 import DeviceGraph, Tuning, harness as H, k_hop_count_device

k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
ns = int(sys.argv[2]) if len(sys.argv) > 2 else 300
eng = {"auto": 0, "single": 1, "lanes": 2}[sys.argv[3] if len(sys.argv) > 3 else "auto"]
W = int(sys.argv[4]) if len(sys.argv) > 4 else 0
rp, ci = H.gen_csr(H.G2)
g = DeviceGraph.from_csr(rp, ci)
if W:
    g.set_tuning(Tuning(lanes_words=W))
seeds = torch.from_numpy(H.pick_seeds(rp, ns, 1).astype(np.int32)).cuda()
counts = torch.zeros(ns, dtype=torch.int64, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    k_hop_count_device(g, seeds.data_ptr(), ns, k, 0, counts.data_ptr(), s, eng)
torch.cuda.synchronize()
print("sum", int(counts.sum()))

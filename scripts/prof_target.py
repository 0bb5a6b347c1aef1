#!/usr/bin/env python3
"""Device-path k-hop launches for ncu: the graph (G2 | G4, generated on the
GPU), the first `nseeds` pick_seeds seeds, `reps` identical launches of
k_hop_count_device (profile one with --launch-skip).

usage: prof_target.py <G2|G4> <k> <nseeds> [lanes_words] [reps]"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1905_01294_b200 import DeviceGraph, Tuning, harness as H, k_hop_count_device  # noqa: E402

gname, k, ns = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
W = int(sys.argv[4]) if len(sys.argv) > 4 else 0
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
g = DeviceGraph.generate(H.SPECS[gname])
rp, _ = g.csr()
if W:
    g.set_tuning(Tuning(lanes_words=W))
seeds = torch.from_numpy(H.pick_seeds(rp, ns, 1).astype(np.int32)).cuda()
counts = torch.zeros(ns, dtype=torch.int64, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for _ in range(reps):
    k_hop_count_device(g, seeds.data_ptr(), ns, k, 0, counts.data_ptr(), s)
torch.cuda.synchronize()
print(gname, "k", k, "seeds", ns, "sum", int(counts.sum()))

import sys, numpy as np
sys.path.insert(0, '.')
from paper_1905_01294_b200 import DeviceGraph, harness as H, k_hop_count_batch
rp, ci = H.gen_csr(H.G2)
g = DeviceGraph.from_csr(rp, ci)
seeds = H.pick_seeds(rp, 300, 1)
for _ in range(2):
    c = k_hop_count_batch(g, seeds, 2, 0)
import torch; torch.cuda.synchronize()
print("DONE", flush=True)

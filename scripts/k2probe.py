import sys, numpy as np
sys.path.insert(0, '.')
from paper_1905_01294_b200 import DeviceGraph, harness as H, k_hop_count_batch
rp, ci = H.gen_csr(H.G2)
g = DeviceGraph.from_csr(rp, ci)
seeds = H.pick_seeds(rp, 300, 1)
for _ in range(3):
    c, st = k_hop_count_batch(g, seeds, 2, 0, stats=True)
print({k: st[k] for k in st if k != 'levels'})
for h in range(3): print(h, st['levels'][h])

"""Child process for test_two_processes_share_one_gpu: the device-resident path
(caller's stream) and the host API path (the library's own non-blocking
stream, fresh workspace) must agree while another process uses the GPU.
Exit code 0 = agreement on every iteration."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_1905_01294_b200 import DeviceGraph, harness as H, k_hop_count_batch, k_hop_count_device  # noqa: E402

spec = H.GraphSpec("S18", scale=18, edge_factor=16, relabel=1)
rp, ci = H.gen_csr(spec)
g = DeviceGraph.from_csr(rp, ci)  # the build frees large temporaries: later allocations reuse them
seeds = H.pick_seeds(rp, 300, 1)
d_seeds = torch.from_numpy(seeds.astype(np.int32)).cuda()
s = torch.cuda.current_stream()
bad = 0
for it in range(10):
    for k in (2, 3):
        d = torch.zeros(len(seeds), dtype=torch.int64, device="cuda")
        k_hop_count_device(g, d_seeds.data_ptr(), len(seeds), k, 0, d.data_ptr(), s.cuda_stream)
        torch.cuda.synchronize()
        if not np.array_equal(d.cpu().numpy().astype(np.uint64), k_hop_count_batch(g, seeds, k, 0)):
            bad += 1
print("mismatches", bad)
sys.exit(1 if bad else 0)

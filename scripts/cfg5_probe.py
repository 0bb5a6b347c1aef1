"""cfg5 timing (G2, 65,536 seeds, LANES auto width): k=3 and k=6, CUDA events, median of 3."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1905_01294_b200 import DeviceGraph, device_stats, harness as H, k_hop_count_device  # noqa: E402

g = DeviceGraph.generate(H.G2)
rp, _ = g.csr()
seeds = H.pick_seeds(rp, 65536, 1)
d_s = torch.from_numpy(seeds.astype(np.int32)).cuda()
d_c = torch.zeros(65536, dtype=torch.int64, device="cuda")
s = torch.cuda.current_stream()
for k in (3, 6):
    k_hop_count_device(g, d_s.data_ptr(), 65536, k, 0, d_c.data_ptr(), s.cuda_stream)
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        k_hop_count_device(g, d_s.data_ptr(), 65536, k, 0, d_c.data_ptr(), s.cuda_stream)
        e1.record(s)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    st = device_stats(g, s.cuda_stream)
    print(f"cfg5 k={k}: {np.median(ts):.1f} ms lanes={st['lanes']} sum={int(d_c.sum())}", flush=True)

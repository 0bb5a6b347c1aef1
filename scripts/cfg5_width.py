"""cfg5 (G2, 65,536 seeds) k = 3 / 6 time per LANES word count W (64·W lanes per batch)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1905_01294_b200 import DeviceGraph, Tuning, harness as H, k_hop_count_device  # noqa: E402

g = DeviceGraph.generate(H.G2)
rp, _ = g.csr()
seeds = H.pick_seeds(rp, 65536, 1)
d_s = torch.from_numpy(seeds.astype(np.int32)).cuda()
d_c = torch.zeros(65536, dtype=torch.int64, device="cuda")
s = torch.cuda.current_stream()
ref = {}
for W in [int(x) for x in sys.argv[1:]] or [8, 4, 2, 1]:
    g.set_tuning(Tuning(lanes_words=W))
    for k in (3, 6):
        k_hop_count_device(g, d_s.data_ptr(), 65536, k, 0, d_c.data_ptr(), s.cuda_stream)
        torch.cuda.synchronize()
        got = d_c.cpu().numpy().copy()
        if k in ref:
            assert (got == ref[k]).all(), (W, k)
        ref[k] = got
        ts = []
        for _ in range(2):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            k_hop_count_device(g, d_s.data_ptr(), 65536, k, 0, d_c.data_ptr(), s.cuda_stream)
            e1.record(s)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        print(f"cfg5 W={W} k={k}: {np.median(ts):.1f} ms", flush=True)

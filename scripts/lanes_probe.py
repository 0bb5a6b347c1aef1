"""LANES engine probe: per-hop device time / scanned entries for the 10-seed
deep configs (cfg3 on G2, cfg4 on G4) under several lane-word widths
(MGK_LANE_BITS), answers cross-checked between widths. Usage:
    python scripts/lanes_probe.py [G2|G4|both] [bits ...]"""
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1905_01294_b200 import DeviceGraph, device_stats, harness as H, k_hop_count_device  # noqa: E402


def run(gname, bits_list, reps=5):
    spec = H.SPECS[gname]
    t = time.time()
    g = DeviceGraph.generate(spec)
    rp, _ = g.csr()
    seeds = H.pick_seeds(rp, 10, 1)
    print(f"{gname}: n={g.nrows} m={g.nnz} ({time.time() - t:.1f}s)", flush=True)
    # the k = 2 group of the schedule (300 seeds, on-chip k2 kernel)
    s300 = torch.from_numpy(H.pick_seeds(rp, 300, 1).astype(np.int32)).cuda()
    c300 = torch.zeros(300, dtype=torch.int64, device="cuda")
    st0 = torch.cuda.current_stream()
    fl = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    k2t = []
    for _ in range(6):
        fl.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st0)
        k_hop_count_device(g, s300.data_ptr(), 300, 2, 0, c300.data_ptr(), st0.cuda_stream)
        e1.record(st0)
        torch.cuda.synchronize()
        k2t.append(e0.elapsed_time(e1))
    print(f"{gname} k2 300 seeds: {np.median(k2t[1:]):.3f} ms sum={int(c300.sum())}", flush=True)
    del fl
    d_seeds = torch.from_numpy(seeds.astype(np.int32)).cuda()
    d_counts = torch.zeros(10, dtype=torch.int64, device="cuda")
    s = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ref = {}
    out = {}
    for bits in bits_list:
        os.environ["MGK_LANE_BITS"] = str(bits)
        for k in (3, 6):
            k_hop_count_device(g, d_seeds.data_ptr(), 10, k, 0, d_counts.data_ptr(), s.cuda_stream)
            torch.cuda.synchronize()
            ans = d_counts.cpu().tolist()
            if k in ref:
                assert ans == ref[k], (gname, bits, k, ans, ref[k])
            ref[k] = ans
            ts = []
            for _ in range(reps):
                flush.fill_(1)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                k_hop_count_device(g, d_seeds.data_ptr(), 10, k, 0, d_counts.data_ptr(), s.cuda_stream)
                e1.record(s)
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            st = device_stats(g, s.cuda_stream)
            diag = os.environ.get("MGK_MS_DIAG") == "1"
            hops = [(h, "pull" if L["pull_runs"] else "push", L["scanned"], round(L["ns"] / 1e3, 1)) +
                    ((round(L["union_edges"] / 1e3, 1), round(L["candidates"] / 1e3, 1),
                      round(L["edges"] / 1e3, 1)) if diag else ())
                    for h, L in enumerate(st["levels"]) if h and L["runs"]]
            out[f"{gname}_b{bits}_k{k}"] = {"ms": float(np.median(ts)), "lanes": st["lanes"], "hops": hops}
            print(f"{gname} bits={bits} k={k}: {np.median(ts):.3f} ms lanes={st['lanes']} hops={hops}", flush=True)
    os.environ.pop("MGK_LANE_BITS", None)
    del g
    torch.cuda.empty_cache()
    return out


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "both"
    bits = [int(b) for b in sys.argv[2:]] or [64, 16]
    # MGK_LANES_UNIFORM=1 in the environment: one direction for all lanes (A/B)
    res = {}
    for gname in (["G2", "G4"] if which == "both" else [which]):
        res.update(run(gname, bits))
    Path("gpurun_out").mkdir(exist_ok=True)
    Path("gpurun_out/lanes_probe.json").write_text(json.dumps(res, indent=1))

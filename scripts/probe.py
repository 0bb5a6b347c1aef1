#!/usr/bin/env python3
"""Exploration probe (not the bench): times engine / lane-width variants on G2
with device-resident seeds and prints per-hop stats as JSON lines."""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1905_01294_b200 import (ENGINE_LANES, ENGINE_SINGLE, DeviceGraph, Tuning, device_stats,
                                   harness as H, k_hop_count_device)


def lc_extra(g, stream):
    import ctypes as C
    from paper_1905_01294_b200 import _lib
    return None


def timeit(g, seeds_np, k, engine, reps=5):
    s = torch.cuda.current_stream()
    d_seeds = torch.from_numpy(seeds_np.astype(np.int32)).cuda()
    d_counts = torch.zeros(len(seeds_np), dtype=torch.int64, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ts = []
    for r in range(reps + 2):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        k_hop_count_device(g, d_seeds.data_ptr(), len(seeds_np), k, 0, d_counts.data_ptr(), s.cuda_stream,
                           engine)
        e1.record(s)
        torch.cuda.synchronize()
        if r >= 2:
            ts.append(e0.elapsed_time(e1))
    st = device_stats(g, s.cuda_stream)
    return float(np.median(ts)), st, d_counts.cpu().numpy()


def main():
    which = sys.argv[1:] or ["cfg2", "cfg3", "cfg5"]
    rp, ci = H.gen_csr(H.G2)
    g = DeviceGraph.from_csr(rp, ci)
    print(json.dumps({"graph": "G2", "n": len(rp) - 1, "m": len(ci)}), flush=True)
    master = H.pick_seeds(rp, 65536, 1)
    if "cfg2" in which:
        g.set_tuning(Tuning())
        for k in (1, 2, 3):
            ms, st, c = timeit(g, master[:300], k, ENGINE_SINGLE)
            print(json.dumps({"cfg": "cfg2", "engine": "single", "k": k, "ms": ms, "qps": 300 / ms * 1e3,
                              "sum": int(c.sum()), "setup_us": st["setup_us"], "cleanup_us": st["cleanup_us"],
                              "hops": [(L["runs"], L["pull_runs"], L["frontier"], L["scanned"], L["candidates"],
                                        round(L["ns"] / 1e3, 1)) for L in st["levels"][1:]]}), flush=True)
        for W in (1, 2, 4, 8):
            g.set_tuning(Tuning(lanes_words=W))
            for k in (1, 2):
                ms, st, c = timeit(g, master[:300], k, ENGINE_LANES)
                print(json.dumps({"cfg": "cfg2", "W": W, "k": k, "ms": ms, "qps": 300 / ms * 1e3,
                                  "sum": int(c.sum()),
                                  "hops": [(L["pull_runs"], L["frontier"], L["vertices"], L["scanned"],
                                            round(L["ns"] / 1e3, 1)) for L in st["levels"][1:]]}),
                      flush=True)
    if "cfg3" in which:
        g.set_tuning(Tuning())
        for k in (3, 6):
            ms, st, c = timeit(g, master[:10], k, ENGINE_SINGLE, reps=3)
            print(json.dumps({"cfg": "cfg3", "engine": "single", "k": k, "ms": ms, "qps": 10 / ms * 1e3,
                              "counts": c.tolist(),
                              "hops": [(L["pull_runs"], L["frontier"], L["edges"], L["scanned"],
                                        L["candidates"], round(L["ns"] / 1e3, 1)) for L in st["levels"][1:]]}),
                  flush=True)
            for W in (1,):
                g.set_tuning(Tuning(lanes_words=W))
                ms, st, c2 = timeit(g, master[:10], k, ENGINE_LANES, reps=3)
                assert (c == c2).all()
                print(json.dumps({"cfg": "cfg3", "engine": f"lanes{W}", "k": k, "ms": ms, "qps": 10 / ms * 1e3,
                                  "hops": [(L["pull_runs"], L["frontier"], L["vertices"], L["scanned"],
                                            round(L["ns"] / 1e3, 1)) for L in st["levels"][1:]]}),
                      flush=True)
            g.set_tuning(Tuning())
    if "cfg5" in which:
        n5 = 4096
        g.set_tuning(Tuning())
        for k in (1, 2):
            ms, st, c = timeit(g, master[:n5], k, ENGINE_SINGLE, reps=2)
            print(json.dumps({"cfg": "cfg5", "engine": "single", "k": k, "seeds": n5, "ms": ms,
                              "qps": n5 / ms * 1e3, "sum": int(c.sum())}), flush=True)
        for W in (1, 2, 4, 8):
            g.set_tuning(Tuning(lanes_words=W))
            for k in (1, 2, 3, 6):
                ms, st, c = timeit(g, master[:n5], k, ENGINE_LANES, reps=2)
                e = sum(L["edges"] for L in st["levels"])
                print(json.dumps({"cfg": "cfg5", "W": W, "k": k, "seeds": n5, "ms": ms, "qps": n5 / ms * 1e3,
                                  "gteps": e / ms / 1e6, "sum": int(c.sum()),
                                  "hops": [(L["pull_runs"], L["vertices"], L["scanned"], round(L["ns"] / 1e3, 1))
                                           for L in st["levels"][1:]]}),
                      flush=True)


if __name__ == "__main__":
    main()

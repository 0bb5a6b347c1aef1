#!/usr/bin/env python3
"""Exploration probe (not the bench): where the host-API (e2e) time of one
k_hop_count_batch call goes, on G2 with cfg2's 300 seeds x k=1,2."""
import ctypes as C
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1905_01294_b200 import DeviceGraph, _lib, harness as H, k_hop_count_batch, k_hop_count_device


def per_call_us(fn, reps=2000):
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    return (time.perf_counter() - t) / reps * 1e6


def main():
    g = DeviceGraph.generate(H.G2, device=0)
    rng = np.random.default_rng(7)
    seeds = rng.integers(0, g.node_count, 300).astype(np.uint64)
    lib = _lib.lib()
    counts = np.empty(300, np.uint64)
    s = torch.cuda.current_stream()
    d_seeds = torch.from_numpy(seeds.astype(np.int32)).cuda()
    d_counts = torch.zeros(300, dtype=torch.int64, device="cuda")
    hs = torch.from_numpy(seeds.astype(np.int32)).pin_memory()
    hc = torch.empty(300, dtype=torch.int64).pin_memory()
    for k in (1, 2):
        r = {}
        r["wrapper"] = per_call_us(lambda: k_hop_count_batch(g, seeds, k, 0))
        r["raw_ctypes"] = per_call_us(lambda: lib.mgk_khop_count_ex(g.handle, seeds.ctypes.data, 300, k, 0, 0,
                                                                     counts.ctypes.data, None))

        def dev_sync():
            k_hop_count_device(g, d_seeds.data_ptr(), 300, k, 0, d_counts.data_ptr(), s.cuda_stream)
            torch.cuda.synchronize()
        r["device_call+sync"] = per_call_us(dev_sync)

        def dev_pipe():
            k_hop_count_device(g, d_seeds.data_ptr(), 300, k, 0, d_counts.data_ptr(), s.cuda_stream)
        r["device_call_pipelined"] = per_call_us(dev_pipe)
        torch.cuda.synchronize()

        def copies():
            d_seeds.copy_(hs, non_blocking=True)
            hc.copy_(d_counts, non_blocking=True)
            torch.cuda.synchronize()
        r["torch_copies+sync"] = per_call_us(copies)

        def tiny():
            d_counts.zero_()
            torch.cuda.synchronize()
        r["tiny_kernel+sync"] = per_call_us(tiny)
        # GPU time of one call when every call is followed by a sync
        ts = []
        for i in range(300):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            k_hop_count_device(g, d_seeds.data_ptr(), 300, k, 0, d_counts.data_ptr(), s.cuda_stream)
            e1.record(s)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        r["gpu_time_synced(med)"] = float(np.median(ts[50:]))
        ts = []
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(301)]
        evs[0].record(s)
        for i in range(300):
            k_hop_count_device(g, d_seeds.data_ptr(), 300, k, 0, d_counts.data_ptr(), s.cuda_stream)
            evs[i + 1].record(s)
        torch.cuda.synchronize()
        ts = [evs[i].elapsed_time(evs[i + 1]) * 1e3 for i in range(300)]
        r["gpu_time_pipelined(med)"] = float(np.median(ts[50:]))
        flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
        for fl in (False, True):
            ts = []
            for i in range(400):
                if fl:
                    flush.fill_(1)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                k_hop_count_batch(g, seeds, k, 0)
                ts.append((time.perf_counter() - t0) * 1e6)
            r[f"bench_loop_flush={fl}"] = float(np.mean(ts[50:]))
            ts = []
            for i in range(400):
                if fl:
                    flush.fill_(1)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                k_hop_count_device(g, d_seeds.data_ptr(), 300, k, 0, d_counts.data_ptr(), s.cuda_stream)
                e1.record(s)
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e3)
            r[f"gpu_flush={fl}"] = float(np.mean(ts[50:]))
        print(f"k={k}: " + "  ".join(f"{a}={b:.1f}us" for a, b in r.items()), flush=True)


if __name__ == "__main__":
    main()

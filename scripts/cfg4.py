#!/usr/bin/env python3
"""BASELINE.json configs[3] (cfg4): the Twitter-shaped R-MAT graph — 2^26 ids,
generated until 1.47B unique directed edges remain, isolated ids dropped and
survivors renumbered — with 300 seeds for k=1,2 and 10 seeds for k=3,6.

Prints one JSON line: generation / upload times, n, m, per-k device time and
q/s / GTEPS (device-resident seeds, CUDA events), and a sampled bit-exact
check against the CPU oracle (oracle/khop_oracle.c; checker only).
usage: cfg4.py [--check-seeds N]"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1905_01294_b200 import DeviceGraph, device_stats, harness as H, k_hop_count_device  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--check-seeds", type=int, default=2)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    res = {"workload": "cfg4", "graph": "G4"}
    t = time.time()
    g = DeviceGraph.generate(H.G4)  # generation, dedup, CSR + CSC on the GPU
    res["gen_build_s"] = time.time() - t
    t = time.time()
    rp, ci = g.csr()  # host copy for pick_seeds and the oracle
    res["download_s"] = time.time() - t
    res["n"], res["m"] = int(len(rp) - 1), int(len(ci))
    print(f"G4: n={res['n']} m={res['m']} built on the GPU in {res['gen_build_s']:.1f}s", file=sys.stderr,
          flush=True)
    res["device_bytes"] = g.device_bytes()
    master = H.pick_seeds(rp, 300, 1)
    s = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    res["k"] = {}
    counts_by_k = {}
    for k, ns in ((1, 300), (2, 300), (3, 10), (6, 10)):
        seeds = master[:ns]
        d_seeds = torch.from_numpy(seeds.astype(np.int32)).cuda()
        d_counts = torch.zeros(ns, dtype=torch.int64, device="cuda")
        k_hop_count_device(g, d_seeds.data_ptr(), ns, k, 0, d_counts.data_ptr(), s.cuda_stream)
        times = []
        for _ in range(args.reps):
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            k_hop_count_device(g, d_seeds.data_ptr(), ns, k, 0, d_counts.data_ptr(), s.cuda_stream)
            e1.record(s)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        st = device_stats(g, s.cuda_stream)
        ms = float(np.median(times))
        edges = sum(L["edges"] for L in st["levels"])
        counts_by_k[k] = d_counts.cpu().numpy().astype(np.uint64)
        res["k"][str(k)] = {"seeds": ns, "ms": ms, "queries_per_s": ns / (ms / 1e3),
                            "gteps": edges / (ms / 1e3) / 1e9, "engine": st["engine"],
                            "hops": [(L["pull_runs"], L["frontier"], L["scanned"], round(L["ns"] / 1e3, 1))
                                     for L in st["levels"][1:] if L["runs"]],
                            "count_sum": int(counts_by_k[k].sum())}
        print(json.dumps({k: res["k"][str(k)]}), file=sys.stderr, flush=True)
    # sampled parity against the CPU oracle (uint64 CSR on the host)
    if args.check_seeds:
        sys.path.insert(0, str(ROOT))
        import oracle
        P = oracle.Port()
        t = time.time()
        rp64, ci64 = rp.astype(np.uint64), ci.astype(np.uint64)
        checked, bad = 0, 0
        for k in (1, 2, 3, 6):
            for i in range(min(args.check_seeds, 10)):
                want = P.khop_count(rp64, ci64, int(master[i]), k, 0)
                got = int(counts_by_k[k][i])
                checked += 1
                bad += want != got
        res["oracle_check"] = {"checked": checked, "mismatches": bad, "seconds": time.time() - t}
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()

#!/usr/bin/env python3
"""Exploration probe (not the bench): SINGLE-engine direction policy on G2 for
many seeds (cfg5 shape) -- auto (Beamer alpha) vs forced push, per k."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parent))
from paper_1905_01294_b200 import DeviceGraph, Tuning, harness as H  # noqa: E402
from probe import timeit  # noqa: E402

rp, ci = H.gen_csr(H.G2)
g = DeviceGraph.from_csr(rp, ci)
master = H.pick_seeds(rp, 65536, 1)
for ns in (300, 4096, 65536):
    for k in (2, 3, 6):
        if k >= 3 and ns > 300:
            continue
        res = []
        for name, t in (("auto", Tuning()), ("a4", Tuning(alpha=4)), ("a8", Tuning(alpha=8)),
                        ("push", Tuning(force_dir=1))):
            g.set_tuning(t)
            ms, st, c = timeit(g, master[:ns], k, 1, reps=2 if ns > 4096 else 5)
            res.append(f"{name}={ms:.3f}ms(sum={int(c.sum())},pull={[L['pull_runs'] for L in st['levels'][1:k+1]]})")
        print(f"ns={ns} k={k}: " + "  ".join(res), flush=True)

#!/usr/bin/env python3
"""The reference's own CPU k_hop_count (oracle/_ref: unmodified matgraph core,
-O3, checks off) on the BASELINE configs that bench.py's reference arm does not
cover, on this host's cores: cfg1 (G1, 300 seeds, k=1,2), cfg3 (G2, 10 seeds,
k=3,6) and cfg5 (G2, a prefix of the 65,536-seed list per k, extrapolated as
SURVEY.md §8(d) prescribes). Prints one JSON line. (Checker / baseline only.)"""
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import oracle  # noqa: E402
from paper_1905_01294_b200 import harness as H  # noqa: E402


def main():
    R = oracle.Ref()
    cores = os.cpu_count() or 1
    out = {"cores": cores, "kind": "reference", "configs": {}}
    for name, spec in (("cfg1", H.G1), ("G2", H.G2)):
        rp, ci = H.gen_csr(spec)
        src, dst = H.csr_to_edges(rp, ci)
        t = time.time()
        g = R.build_bench_graph(src, dst, len(rp) - 1)
        build_s = time.time() - t
        if name == "cfg1":
            seeds = H.pick_seeds(rp, 300, 1)
            sec = {"build_s": build_s}
            for k in (1, 2):
                _, el = g.k_hop_count_many(seeds, k, 0, threads=cores)
                sec[f"k{k}"] = {"seeds": 300, "s": el, "queries_per_s": 300 / el}
            out["configs"]["cfg1"] = sec
            continue
        master = H.pick_seeds(rp, 65536, 1)
        out["configs"]["cfg3"] = {}
        for k in (3, 6):
            _, el = g.k_hop_count_many(master[:10], k, 0, threads=cores)
            out["configs"]["cfg3"][f"k{k}"] = {"seeds": 10, "s": el, "queries_per_s": 10 / el}
        sec = {"note": "prefix of the cfg5 seed list, all host threads; q/s extrapolates to 65,536 seeds"}
        for k, n in ((1, 65536), (2, 4096), (3, 64), (6, 64)):
            _, el = g.k_hop_count_many(master[:n], k, 0, threads=cores)
            sec[f"k{k}"] = {"seeds": n, "s": el, "queries_per_s": n / el,
                            "extrapolated_s_for_65536": el * 65536 / n}
        out["configs"]["cfg5"] = sec
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()

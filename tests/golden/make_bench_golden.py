"""Golden vectors for the BASELINE.json bench configs (cfg2-cfg5), made here
where the reference builds, committed as tests/golden/bench_pins.json.

    make -C oracle all && python tests/golden/make_bench_golden.py [--no-g4]

What is pinned, and by what:

* the bench graphs G2 (2^22 ids, 67,108,864 unique edges) and G4 (2^26 ids,
  1.47B unique edges): n, m and the SHA-256 of the uint32 CSR produced by the
  oracle's independent restatement of the generator (oracle/bench_oracle.c
  orc_gen_bench_csr). The product's host and GPU generators must hash equal.
* the seeds: pick_seeds (bench.cpp:200-218) as restated by
  orc_pick_seeds_u32 (pinned to the reference's own pick_seeds by
  tests/test_bench_oracle.py), the 300-seed prefix and the SHA-256 of the
  65,536-seed cfg5 list.
* the counts FROM THE REFERENCE ITSELF: the unmodified reference core
  (oracle/_ref) runs k_hop_frontier's vxm / ewise_union loop
  (execute.cpp:347-375) over a SparseMatrix::from_parts of the same CSR
  (sparse.cpp:101-114; the PropertyGraph wrapper is bypassed because
  build_bench_graph of G4 needs ~70 GB):
    cfg2  300 seeds x k=1,2   exact + cumulative
    cfg3   10 seeds x k=3,6   exact + cumulative
    cfg4  300 seeds x k=1,2 and 20 seeds x k=3,6, exact + cumulative
* cfg5: per-level frontier sizes |F_1|..|F_6| (exact count at every k; the
  cumulative count is their prefix sum) of 1,536 seeds of the 65,536-seed list
  — all of W=8 lane batches 0, 64 and 127 (512 seeds each) — from the C
  oracle's bulk BFS (orc_khop_many), cross-checked against the reference on
  the first 32 seeds of each batch here.

The GPU box never runs this script; tests/test_gpu_configs.py reads the JSON.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import oracle  # noqa: E402

OUT = Path(__file__).resolve().parent / "bench_pins.json"

# BASELINE.json graph recipes (same numbers as paper_1905_01294_b200.harness)
G2 = dict(scale=22, edge_factor=16, target_unique=67_108_864, relabel=2)
G4 = dict(scale=26, edge_factor=16, target_unique=1_470_000_000, relabel=2)
CFG5_BATCHES = (0, 64, 127)  # W=8: 512 seeds per batch
CFG5_BATCH = 512


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def ref_counts(M, seeds, ks, threads):
    """{k: {"exact": [...], "cumulative": [...]}} from the reference matrix route."""
    out = {}
    for k in ks:
        ent = {}
        for mode, name in ((0, "exact"), (1, "cumulative")):
            t = time.time()
            c, _ = M.khop_jobs(seeds, np.full(len(seeds), k, np.uint32), mode, threads)
            ent[name] = [int(x) for x in c]
            log(f"  reference k={k} {name}: {len(seeds)} seeds in {time.time() - t:.1f}s")
        out[str(k)] = ent
    return out


def graph_pins(P, R, spec, name, plan, threads, cfg5=False):
    t = time.time()
    rp, ci = P.gen_bench_csr(**spec)
    log(f"{name}: n={len(rp) - 1} m={len(ci)} generated in {time.time() - t:.1f}s")
    g = {"n": int(len(rp) - 1), "m": int(len(ci)), "spec": spec, "csr_sha256": sha(rp, ci),
         "max_out_degree": int(np.diff(rp.astype(np.int64)).max())}
    master = P.pick_seeds_u32(rp, 65536 if cfg5 else 300, 1)
    g["seeds300"] = [int(s) for s in master[:300]]
    t = time.time()
    M = R.matrix(rp, ci)
    log(f"{name}: reference from_parts in {time.time() - t:.1f}s")
    g["ref"] = {}
    for label, nseeds, ks in plan:
        g["ref"][label] = {"nseeds": nseeds, "counts": ref_counts(M, master[:nseeds], ks, threads)}
    # the C oracle agrees with the reference on every pinned count
    for label, nseeds, ks in plan:
        for k in ks:
            ex, cu = P.khop_many(rp, ci, master[:nseeds], k)
            r = g["ref"][label]["counts"][str(k)]
            assert ex.tolist() == r["exact"] and cu.tolist() == r["cumulative"], (name, label, k)
    if cfg5:
        g["seeds65536_sha256"] = sha(master)
        idx = np.concatenate([np.arange(b * CFG5_BATCH, (b + 1) * CFG5_BATCH) for b in CFG5_BATCHES])
        t = time.time()
        _, _, edges, levels = P.khop_many(rp, ci, master[idx], 6, work=True)
        log(f"{name}: cfg5 sample levels for {len(idx)} seeds in {time.time() - t:.1f}s")
        g["cfg5"] = {"batches": list(CFG5_BATCHES), "batch_seeds": CFG5_BATCH,
                     "levels": [[int(x) for x in row[1:]] for row in levels],
                     "edges_k6": [int(x) for x in edges]}
        # reference cross-check on the first 32 seeds of each sampled batch
        for b in range(len(CFG5_BATCHES)):
            sel = master[idx[b * CFG5_BATCH:b * CFG5_BATCH + 32]]
            for k in (2, 3, 6):
                c, _ = M.khop_jobs(sel, np.full(len(sel), k, np.uint32), 0, threads)
                want = [row[k] for row in levels[b * CFG5_BATCH:b * CFG5_BATCH + 32]]
                assert [int(x) for x in c] == [int(x) for x in want], (b, k)
    del M
    return g


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--no-g4", action="store_true")
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    args = ap.parse_args()
    P, R = oracle.Port(), oracle.Ref()
    pins = json.loads(OUT.read_text()) if OUT.exists() else {}
    pins["_generated_by"] = "tests/golden/make_bench_golden.py (oracle/_ref + oracle/liboracle.so)"
    pins["G2"] = graph_pins(P, R, G2, "G2", [("cfg2", 300, (1, 2)), ("cfg3", 10, (3, 6))], args.threads,
                            cfg5=True)
    OUT.write_text(json.dumps(pins, separators=(",", ":")))
    if not args.no_g4:
        pins["G4"] = graph_pins(P, R, G4, "G4", [("cfg4_k12", 300, (1, 2)), ("cfg4_k36", 20, (3, 6))],
                                args.threads)
        OUT.write_text(json.dumps(pins, separators=(",", ":")))
    log(f"wrote {OUT}")


if __name__ == "__main__":
    main()

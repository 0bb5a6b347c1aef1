#!/usr/bin/env python3
"""k-hop count benchmark (BASELINE.json metric) — one JSON line on rank 0.

Headline workload (N=1): BASELINE.json configs[3] ("cfg4"), the largest
single-GPU config: the Twitter-shaped R-MAT graph G4 (a=.57 b=.19 c=.19
d=.05 over 2^26 ids until 1,470,000,000 unique directed edges remain,
isolated ids dropped and survivors renumbered: n = 35,559,419) and the
reference harness's default schedule (proj/tools/matgraph.cpp:20-21):
k = 1, 2, 3, 6 with 300 / 300 / 10 / 10 seeds, the 10-seed sections being
prefixes of the 300-seed pick_seeds list (bench.cpp:200-218, 311-343). A step
is that whole schedule, 620 exact k-hop counts. Metric: queries/s, plus GTEPS
(push-equivalent edges).

Multi-GPU (torchrun, or `--gpus N` which re-launches itself under torchrun):
every rank generates its own replica of G4 on its GPU and runs its own
schedule on a disjoint 300-seed shard of one master list (weak scaling, no
collective on the data path); max-over-ranks device time.

Arms:
  default           the sm_100a engine (libmgk.so). `value`: device-resident
                    seeds / counts, one mgk_khop_count_device_schedule call per
                    step, CUDA events on the launch stream, L2 flushed between
                    steps (outside the events). `e2e`: the public host API
                    (k_hop_count_schedule: host uint64 seeds in, host counts
                    out). Every answer is checked against the CPU oracle before
                    timing (and, on rank 0, against the reference's own counts).
  --impl reference  the reference's own CPU k-hop loop (oracle/_ref: the
                    unmodified matgraph core's vxm / ewise_union, execute.cpp:
                    347-375, over SparseMatrix::from_parts of G4 — the
                    PropertyGraph wrapper is bypassed because build_bench_graph
                    of 1.47B edges needs ~70 GB) on all host
                    threads. Input preparation uses the C oracle's generator and
                    pick_seeds restatement (oracle/bench_oracle.c); this arm
                    never loads the product library.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

# BASELINE.json graph recipes (same numbers as paper_1905_01294_b200.harness; kept
# here so the reference arm never imports the product package)
G2 = dict(name="G2", scale=22, edge_factor=16, target_unique=67_108_864, relabel=2)
G4 = dict(name="G4", scale=26, edge_factor=16, target_unique=1_470_000_000, relabel=2)
RMAT = [0.57, 0.19, 0.19, 0.05]
SCHEDULE = {"cfg4": (G4, (1, 2, 3, 6), (300, 300, 10, 10)),   # matgraph.cpp:20-21 on G4
            "cfg2": (G2, (1, 2), (300, 300)),                  # BASELINE configs[1]
            "cfg3": (G2, (3, 6), (10, 10))}                    # BASELINE configs[2]
SEEDS_PER_RANK = 300
METRIC = "k-hop count queries/s (k=1,2,3,6 x 300/300/10/10 seeds, exact; reference default schedule)"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text()), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return {"hbm_gbs": 6650.0}, "fallback (B200_PROFILING.md)"


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def workload_config(name: str, world: int, n: int | None = None, m: int | None = None) -> dict:
    """The `config` object — identical keys and values in both arms."""
    spec, ks, ns = SCHEDULE[name]
    return {"workload": name, "graph": {"name": spec["name"], "ids": f"2^{spec['scale']} renumbered",
                                        "unique_edges": spec["target_unique"], "n": n, "m": m, "rmat": RMAT},
            "schedule": {"ks": list(ks), "seeds_per_k": list(ns), "mode": "exact",
                         "source": "proj/tools/matgraph.cpp:20-21 (bench default)" if name == "cfg4" else "BASELINE.json"},
            "seeds_per_rank": max(ns), "ranks": world,
            "l2": "flushed between steps (256 MiB write outside the events); the graph (>= 0.56 GB) exceeds L2"}


class ClockSampler:
    """NVML clocks + throttle reasons sampled every 2 ms in a thread during the
    timed region (a 50 ms nvidia-smi poll misses short regions)."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, index: int, period_s: float = 0.002):
        self.index, self.period = index, period_s
        self.sm, self.reasons, self.max = [], set(), None
        self._stop = threading.Event()
        self.err = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception as e:  # no NVML: report it, never fail the bench
            self.err = str(e)[:120]
            self.nv = None
        return self

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.sm.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                get = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                    nv.nvmlDeviceGetCurrentClocksThrottleReasons
                r = get(self.h)
                for name, bit in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception as e:
                self.err = str(e)[:120]
                return
            time.sleep(self.period)

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join(timeout=2)

    def summary(self):
        out = {"sm_mhz": float(np.median(self.sm)) if self.sm else None, "sm_max_mhz": self.max,
               "reasons": sorted(self.reasons), "samples": len(self.sm), "source": "NVML, 2 ms period"}
        if self.err:
            out["error"] = self.err
        return out


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def seed_shard(master, rank: int, world: int, per_rank: int):
    """Rank r's disjoint shard of the master seed list (weak scaling)."""
    if len(master) < per_rank * world:
        raise ValueError(f"master list of {len(master)} seeds cannot give {world} shards of {per_rank}")
    return master[rank * per_rank:(rank + 1) * per_rank]


# ---- SURVEY.md §8(d) algorithmic bytes ----------------------------------------------
def single_source_bytes(st: dict, nseeds: int) -> float:
    """B = 4 E + 12 sum_{l<L} |F_l| + 4 sum_{1<=l<=L} |F_l| summed over seeds,
    from the engine's per-hop counters (edges = push-equivalent E, frontier =
    sum of |F_l|). F_0 = the seeds. A level after an early exit has |F| = 0."""
    lv = st["levels"]
    hops = [h for h in range(1, len(lv)) if lv[h]["runs"]]
    if not hops:
        return 0.0
    last = hops[-1]
    E = sum(lv[h]["edges"] for h in hops)
    expanded = nseeds + sum(lv[h]["frontier"] for h in hops if h < last)
    written = sum(lv[h]["frontier"] for h in hops)
    return 4.0 * E + 12.0 * expanded + 4.0 * written


def lanes_bytes(st: dict, n: int) -> float:
    """64-lane mode: per expanded level l, U_l = vertices with
    a non-zero frontier word: 4 sum_{v in U_l} outdeg(v) + 12 |U_l| + 24 W n
    (three streaming passes over n W-word state words), per batch. The
    counters are summed over batches: union_edges of hop h = sum of outdeg
    over U_{h-1}, vertices of hop h-1 = |U_{h-1}|, runs = batches expanded.""" 
    lv = st["levels"]
    W = max(1, st["lanes"] // 64)
    total = 0.0
    for h in range(1, len(lv)):
        if not lv[h]["runs"]:
            continue
        U = lv[h - 1]["vertices"]  # summed over the batches that expanded
        total += 4.0 * lv[h]["union_edges"] + 12.0 * U + 24.0 * W * n * lv[h]["runs"]
    return total


def algo_bytes(st: dict, nseeds: int, n: int) -> float:
    return lanes_bytes(st, n) if st["engine"] == "lanes" else single_source_bytes(st, nseeds)


def push_edges(st: dict) -> int:
    return int(sum(L["edges"] for L in st["levels"][1:] if L["runs"]))


# ---- our arm --------------------------------------------------------------------------
class Arm:
    """One workload on one rank: device graph, seeds, oracle-checked answers."""

    def __init__(self, name, torch, local, rank, world, graph=None, host_csr=None):
        from paper_1905_01294_b200 import DeviceGraph, harness as H
        self.name, self.torch, self.rank, self.world = name, torch, rank, world
        spec, self.ks, self.ns = SCHEDULE[name]
        hspec = H.SPECS[spec["name"]]
        t = time.time()
        self.g = graph if graph is not None else DeviceGraph.generate(hspec, device=local)
        self.gen_s = time.time() - t
        t = time.time()
        self.rp, self.ci = host_csr if host_csr is not None else self.g.csr()
        self.n, self.m = int(self.g.nrows), int(self.g.nnz)
        master = H.pick_seeds(self.rp, SEEDS_PER_RANK * world, 1)
        self.master = master
        self.seeds = seed_shard(master, rank, world, SEEDS_PER_RANK)  # the longest section's seeds
        log(f"[rank {rank}] {name}: {spec['name']} n={self.n} m={self.m} generated on the GPU in "
            f"{self.gen_s:.1f}s, CSR downloaded in {time.time() - t:.1f}s")
        self.d_seeds = torch.from_numpy(self.seeds.astype(np.int32)).cuda()
        self.d_out = torch.zeros(sum(self.ns), dtype=torch.int64, device="cuda")
        self.stream = torch.cuda.current_stream()

    def step(self, ns=None, ks=None, out=None):
        from paper_1905_01294_b200 import k_hop_count_device_schedule
        k_hop_count_device_schedule(self.g, self.d_seeds.data_ptr(), list(ns or self.ns), list(ks or self.ks), 0,
                                    (out if out is not None else self.d_out).data_ptr(), self.stream.cuda_stream)

    def answers(self):
        from paper_1905_01294_b200 import device_check
        device_check(self.g, self.stream.cuda_stream)
        out = self.d_out.cpu().numpy().astype(np.uint64)
        res, off = {}, 0
        for k, n in zip(self.ks, self.ns):
            res[k] = out[off:off + n]
            off += n
        return res

    def groups(self):
        """The schedule's launch groups: consecutive sections with one seed count
        share a launch (mgk_khop_count_device_schedule)."""
        gs, a = [], 0
        while a < len(self.ks):
            b = a + 1
            while b < len(self.ks) and self.ns[b] == self.ns[a]:
                b += 1
            gs.append((tuple(self.ns[a:b]), tuple(self.ks[a:b])))
            a = b
        return gs


def oracle_check(arm: Arm, got: dict, pins: dict | None) -> dict:
    """Every answer of this rank's schedule against the C oracle's BFS
    (oracle/bench_oracle.c orc_khop_many on the host copy of the same CSR, all
    host threads), and on rank 0 also against the reference's own counts
    pinned in tests/golden/bench_pins.json when the generated graph hashes
    equal to the pinned one. Raises on any mismatch."""
    import oracle
    P = oracle.Port()
    t = time.time()
    checked = mism = 0
    deepest = {}
    for k, n in zip(arm.ks, arm.ns):
        deepest[n] = max(deepest.get(n, 0), k)
    levels = {}
    for n, kmax in deepest.items():
        _, _, _, lv = P.khop_many(arm.rp, arm.ci, arm.seeds[:n], kmax, work=True)
        levels[n] = lv
    for k, n in zip(arm.ks, arm.ns):
        want = levels[n][:, k]
        bad = int((got[k] != want).sum())
        checked += n
        mism += bad
    out = {"checked": checked, "mismatches": mism, "against": ["C oracle BFS (orc_khop_many) on the same CSR"],
           "oracle_s": round(time.time() - t, 1)}
    gname = SCHEDULE[arm.name][0]["name"]
    if pins and gname in pins and arm.rank == 0 and arm.world == 1:
        p = pins[gname]
        if arm.n == p["n"] and arm.m == p["m"] and sha(arm.rp, arm.ci) == p["csr_sha256"]:
            rc = 0
            for label, ent in p["ref"].items():
                for kk, c in ent["counts"].items():
                    k = int(kk)
                    if k in got:
                        w = np.array(c["exact"][:len(got[k])], np.uint64)
                        mism += int((got[k][:len(w)] != w).sum())
                        rc += len(w)
            out["against"].append(f"reference counts (tests/golden/bench_pins.json from oracle/_ref): {rc} answers")
            out["reference_checked"] = rc
            out["graph_sha256_matches_pin"] = True
        else:
            out["graph_sha256_matches_pin"] = False
            mism += 1  # the generated graph is not the pinned one: fail loudly
    out["mismatches"] = mism
    if mism:
        raise AssertionError(f"{arm.name}: {mism} answers differ from the oracle / reference: {out}")
    return out


def time_steps(arm: Arm, flush, steps: int, warmup: int, dist=None):
    torch = arm.torch
    for _ in range(warmup):
        flush.fill_(1)
        arm.step()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    ms = []
    for _ in range(steps):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(arm.stream)
        arm.step()
        e1.record(arm.stream)
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    if dist is not None:
        dist.barrier()
    return ms


def group_profile(arm: Arm, flush, reps: int):
    """Each launch group of the schedule on its own (CUDA events on the launch
    stream): per-group time, the engine's counters, §8(d) bytes and GTEPS."""
    from paper_1905_01294_b200 import device_stats
    torch = arm.torch
    pk, pk_src = peaks()
    res = []
    out = torch.zeros(sum(arm.ns), dtype=torch.int64, device="cuda")
    for ns, ks in arm.groups():
        times = []
        for _ in range(reps):
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(arm.stream)
            arm.step(ns, ks, out)
            e1.record(arm.stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        st = device_stats(arm.g, arm.stream.cuda_stream)
        ms = float(np.mean(times))
        kern = ("k2_kernel" if st["path"] == "smem_k2" else
                f"ms_kernel<W={max(1, st['lanes'] // 64)}>" if st["engine"] == "lanes" else "fr_kernel + fr_finish")
        b = algo_bytes(st, ns[0], arm.n)
        res.append({"ks": list(ks), "seeds": ns[0], "kernel": kern, "engine": st["engine"], "lanes": st["lanes"],
                    "launches": st["launches"], "ms_per_call": ms, "algo_bytes": b,
                    "achieved_GBps": b / (ms / 1e3) / 1e9, "frac_of_peak": b / (ms / 1e3) / 1e9 / pk["hbm_gbs"],
                    "push_equiv_edges": push_edges(st), "gteps": push_edges(st) / (ms / 1e3) / 1e9,
                    "hops": [{"hop": h, "dir": "pull" if L["pull_runs"] else "push", "frontier": L["frontier"],
                              "vertices": L["vertices"], "edges": L["edges"], "union_edges": L["union_edges"],
                              "scanned": L["scanned"], "us": L["ns"] / 1e3}
                             for h, L in enumerate(st["levels"]) if h and L["runs"]]})
    return res


def e2e_steps(arm: Arm, flush, steps: int, warmup: int, dist=None):
    """The public host API (k_hop_count_schedule): host uint64 seeds in, host
    counts out, one call per step, wall clock."""
    from paper_1905_01294_b200 import k_hop_count_schedule
    torch = arm.torch
    seeds = np.ascontiguousarray(arm.seeds, np.uint64)
    for _ in range(warmup):
        k_hop_count_schedule(arm.g, seeds, arm.ns, arm.ks, 0)
    if dist is not None:
        dist.barrier()
    ms = []
    got = None
    for _ in range(steps):
        flush.fill_(1)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        got = k_hop_count_schedule(arm.g, seeds, arm.ns, arm.ks, 0)
        ms.append((time.perf_counter() - t0) * 1e3)
    return ms, got


def cpu_baseline_cfg4(arm: Arm, budget_deep: int = 2) -> dict:
    """The reference's own k-hop loop (oracle/_ref, matrix route) on this host,
    all threads, on a BOUNDED sample of the schedule: all 300 k=1 and 300 k=2
    queries and the first `budget_deep` seeds at k=3 and k=6; the schedule's
    q/s is extrapolated from the sample (deep sections x 10/budget_deep) at
    ideal packing on the host threads. The sample's answers are also compared
    with ours (parity)."""
    import oracle
    cores = os.cpu_count() or 1
    try:
        R = oracle.Ref()
    except Exception as e:
        return {"unavailable": f"oracle/_ref not built: {str(e)[:100]}"}
    t = time.time()
    M = R.matrix(arm.rp, arm.ci)
    prep = time.time() - t
    res, per = {}, {}
    for k, n in zip(arm.ks, arm.ns):
        n_s = n if n > 10 else min(n, budget_deep)
        s = arm.seeds[:n_s]
        th = cores if n_s > 10 else n_s
        c, el = M.khop_jobs(s, np.full(len(s), k, np.uint32), 0, threads=th)
        res[k] = c
        per[k] = {"seeds": int(n_s), "wall_s": el, "threads": th,
                  "core_s_per_query": el * min(th, n_s) / n_s}
    # extrapolated schedule wall time on `cores` threads (ideal packing of the
    # 10-seed deep queries; k=1 / k=2 measured as run)
    deep = sum(per[k]["core_s_per_query"] * n for k, n in zip(arm.ks, arm.ns) if n <= 10)
    deep_long = max([per[k]["core_s_per_query"] for k, n in zip(arm.ks, arm.ns) if n <= 10] or [0.0])
    wall = sum(per[k]["wall_s"] for k, n in zip(arm.ks, arm.ns) if n > 10) + max(deep / cores, deep_long)
    core_total = sum(per[k]["core_s_per_query"] * n for k, n in zip(arm.ks, arm.ns))
    del M
    return {"value": sum(arm.ns) / wall, "unit": "queries/s", "cores": cores, "kind": "reference",
            "sample": f"oracle/_ref matrix route (vxm/ewise_union loop of execute.cpp:347-375 over from_parts of "
                      f"the same G4 CSR): all 300 k=1 and 300 k=2 queries, first {budget_deep} seeds at k=3 and k=6; "
                      f"schedule wall time extrapolated at ideal packing on {cores} threads",
            "single_core": {"value": sum(arm.ns) / core_total, "unit": "queries/s", "cores": 1},
            "per_k": {str(k): v for k, v in per.items()}, "from_parts_s": prep,
            "_answers": res}


def cpu_baseline_g2(arm: Arm) -> dict:
    """cfg2 (G2, 300 x k=1,2): the reference's own k-hop loop (oracle/_ref,
    matrix route as for cfg4) over the same CSR, all host threads, repeated
    passes of the whole workload for ~8 s."""
    import oracle
    cores = os.cpu_count() or 1
    try:
        R = oracle.Ref()
    except Exception as e:
        return {"unavailable": f"oracle/_ref not built: {str(e)[:100]}"}
    t = time.time()
    M = R.matrix(arm.rp, arm.ci)
    prep = time.time() - t
    passes, el, res = 0, 0.0, {}
    while el < 8.0 and passes < 20:
        for k in arm.ks:
            c, e = M.khop_jobs(arm.seeds, np.full(len(arm.seeds), k, np.uint32), 0, threads=cores)
            res[k] = c
            el += e
        passes += 1
    q = passes * len(arm.seeds) * len(arm.ks)
    t1 = sum(M.khop_jobs(arm.seeds, np.full(len(arm.seeds), k, np.uint32), 0, threads=1)[1] for k in arm.ks)
    return {"value": q / el, "unit": "queries/s", "cores": cores, "kind": "reference",
            "sample": f"{passes} pass(es) of 300 seeds x k=1,2 exact on oracle/_ref (matrix route over the same "
                      f"G2 CSR), {el:.1f}s",
            "single_core": {"value": len(arm.seeds) * len(arm.ks) / t1, "unit": "queries/s", "cores": 1},
            "from_parts_s": prep, "_answers": res}


def secondary(name, torch, local, rank, world, dist, flush, steps, warmup, graph=None, host_csr=None, cpu=True):
    """A further BASELINE config on the same rank (cfg2 / cfg3 on G2): value,
    e2e, per-group roofline, oracle parity (+ reference parity for cfg2)."""
    arm = Arm(name, torch, local, rank, world, graph=graph, host_csr=host_csr)
    for _ in range(2):
        arm.step()
    got = arm.answers()
    parity = oracle_check(arm, got, load_pins())
    ms = time_steps(arm, flush, steps, warmup, dist)
    t = max_over_ranks(torch, dist, float(np.sum(ms)))
    e2e_ms, _ = e2e_steps(arm, flush, steps, max(3, warmup), dist)
    te = max_over_ranks(torch, dist, float(np.sum(e2e_ms)))
    groups = group_profile(arm, flush, min(steps, 20))
    q = sum(arm.ns) * world
    out = {"value": q * steps / (t / 1e3), "unit": "queries/s", "ms_per_step": t / steps,
           "config": workload_config(name, world, arm.n, arm.m), "parity": parity,
           "gteps": sum(gr["push_equiv_edges"] for gr in groups) * world / (sum(gr["ms_per_call"] for gr in groups) / 1e3) / 1e9,
           "e2e": {"value": q * steps / (te / 1e3), "unit": "queries/s"}, "groups": groups}
    if cpu and name == "cfg2" and rank == 0 and world == 1:
        cb = cpu_baseline_g2(arm)
        ans = cb.pop("_answers", {})
        if ans:
            bad = sum(int((np.asarray(ans[k], np.uint64) != got[k]).sum()) for k in arm.ks)
            parity["against"].append(f"the cpu_baseline's own reference answers: {sum(len(ans[k]) for k in ans)}")
            if bad:
                raise AssertionError(f"cfg2: {bad} answers differ from the reference's k_hop_count")
        out["cpu_baseline"] = cb
    return out, arm


def cfg5_section(arm2: Arm, flush, dist):
    """BASELINE configs[4]: 65,536 seeds in 64-lane words, k=1,2,3,6, seed
    batches split across ranks (strong scaling of a fixed 65,536-seed list);
    aggregate q/s and GTEPS. Answers of batch 0's seeds checked against the
    oracle (the full check is tests/test_gpu_configs.py)."""
    from paper_1905_01294_b200 import device_stats, harness as H, k_hop_count_device
    import oracle
    torch = arm2.torch
    world, rank = arm2.world, arm2.rank
    master = H.pick_seeds(arm2.rp, 65536, 1)
    seeds = cfg5_shard(master, rank, world)
    d_seeds = torch.from_numpy(seeds.astype(np.int32)).cuda()
    d_counts = torch.zeros(len(seeds), dtype=torch.int64, device="cuda")
    sp = arm2.stream.cuda_stream
    P = oracle.Port()
    _, _, _, lv = P.khop_many(arm2.rp, arm2.ci, seeds[:64], 6, work=True)
    out = {"seeds": 65536, "seeds_per_rank": int(len(seeds)), "scaling": "strong (fixed 65,536-seed list)", "k": {}}
    for k in (1, 2, 3, 6):
        k_hop_count_device(arm2.g, d_seeds.data_ptr(), len(seeds), k, 0, d_counts.data_ptr(), sp)
        torch.cuda.synchronize()
        got = d_counts[:64].cpu().numpy().astype(np.uint64)
        if not np.array_equal(got, lv[:, k]):
            raise AssertionError(f"cfg5 k={k}: answers differ from the oracle")
        times = []
        for _ in range(3):
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(arm2.stream)
            k_hop_count_device(arm2.g, d_seeds.data_ptr(), len(seeds), k, 0, d_counts.data_ptr(), sp)
            e1.record(arm2.stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        st = device_stats(arm2.g, sp)
        ms = max_over_ranks(torch, dist, float(np.median(times)))
        e = push_edges(st)
        b = algo_bytes(st, len(seeds), arm2.n)
        tot_e = sum_over_ranks(torch, dist, float(e))
        pk, _ = peaks()
        out["k"][str(k)] = {"ms": ms, "queries_per_s": 65536 / (ms / 1e3), "gteps": tot_e / (ms / 1e3) / 1e9,
                            "engine": st["engine"], "lanes_per_batch": st["lanes"],
                            "algo_bytes_rank": b, "frac_of_peak_rank": b / (float(np.median(times)) / 1e3) / 1e9 / pk["hbm_gbs"],
                            "parity": "batch-0 seeds (64) == oracle"}
    return out


def _reduce(torch, dist, x: float, op) -> float:
    if dist is None:
        return x
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=op)
    return float(t[0])


def max_over_ranks(torch, dist, x: float) -> float:
    """The job's time: the slowest rank's (device-timed) figure."""
    return _reduce(torch, dist, x, dist.ReduceOp.MAX if dist is not None else None)


def sum_over_ranks(torch, dist, x: float) -> float:
    return _reduce(torch, dist, x, dist.ReduceOp.SUM if dist is not None else None)


def cfg5_shard(master, rank: int, world: int):
    """cfg5 (strong scaling): rank r's contiguous share of the 65,536-seed list,
    whole 64-lane batches where the split allows (1,024 batches / world)."""
    per = len(master) // world
    extra = len(master) - per * world
    a = rank * per + min(rank, extra)
    return master[a:a + per + (1 if rank < extra else 0)]


def load_pins():
    p = ROOT / "tests" / "golden" / "bench_pins.json"
    try:
        return json.loads(p.read_text())
    except Exception:
        return None


def traffic_of(key: str):
    tf = ROOT / "profiles" / "traffic.json"
    try:
        return json.loads(tf.read_text()).get(key)
    except Exception:
        return None


def run_ours(args):
    import torch
    import torch.distributed as dist_mod

    rank, local, world = dist_env()
    dry = os.environ.get("MGK_BENCH_DRYRUN") == "1"  # gloo + shared devices: functional check only
    if dry:
        local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        if dry:
            dist_mod.init_process_group("gloo")
        else:
            dist_mod.init_process_group("nccl", device_id=torch.device("cuda", local))
        dist = dist_mod
    flush = torch.empty(256 * 2**20, dtype=torch.uint8, device="cuda")  # > 126 MB L2
    name = args.workload
    pins = load_pins()

    # ---- headline ---------------------------------------------------------------------
    arm = Arm(name, torch, local, rank, world)
    for _ in range(2):
        arm.step()
    got = arm.answers()
    cpu = None
    if name == "cfg4" and rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline_cfg4(arm)
    parity = oracle_check(arm, got, pins)
    if cpu and "_answers" in cpu:
        ans = cpu.pop("_answers")
        bad = sum(int((np.asarray(ans[k], np.uint64) != got[k][:len(ans[k])]).sum()) for k in ans)
        parity["against"].append(f"the cpu_baseline's own reference answers: {sum(len(a) for a in ans.values())}")
        if bad:
            raise AssertionError(f"{bad} answers differ from the reference's own k-hop loop")

    sampler = ClockSampler(local)
    with sampler:
        ms = time_steps(arm, flush, args.steps, args.warmup, dist)
        e2e_ms, e2e_got = e2e_steps(arm, flush, args.steps, max(3, args.warmup), dist)
    clocks = sampler.summary()
    for k, x in zip(arm.ks, e2e_got):
        if not np.array_equal(x, got[k]):
            raise AssertionError(f"e2e answers for k={k} differ from the device path")
    total_ms = max_over_ranks(torch, dist, float(np.sum(ms)))
    e2e_total = max_over_ranks(torch, dist, float(np.sum(e2e_ms)))
    groups = group_profile(arm, flush, min(args.steps, 10))

    # ---- secondary configs on G2 (every rank takes part) ---------------------------------
    extras = {}
    if not args.no_extras:
        arm2 = None
        for nm in ("cfg2", "cfg3"):
            if nm == name:
                continue
            sec, a = secondary(nm, torch, local, rank, world, dist, flush, args.steps, args.warmup,
                               graph=arm2.g if arm2 else None, host_csr=(arm2.rp, arm2.ci) if arm2 else None,
                               cpu=not args.no_cpu)
            extras[nm] = sec
            arm2 = arm2 or a
        if arm2 is not None:
            extras["cfg5"] = cfg5_section(arm2, flush, dist)

    if rank != 0:
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()
        return

    q_per_step = sum(arm.ns) * world
    value = q_per_step * args.steps / (total_ms / 1e3)
    dom = max(groups, key=lambda g: g["ms_per_call"])
    pk, pk_src = peaks()
    edges_step = sum(g["push_equiv_edges"] for g in groups) * world
    tr = traffic_of(f"{name}_{dom['kernel'].split('<')[0]}")
    line = {
        "metric": METRIC if name == "cfg4" else f"k-hop count queries/s ({name})",
        "value": value,
        "unit": "queries/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": total_ms / args.steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u32 vertex ids, u64 lane words (integer)",
        "data": "synthetic R-MAT, BASELINE.json configs shape (seeded; stands in for the paper's Twitter / Graph500 graphs)",
        "config": workload_config(name, world, arm.n, arm.m),
        "gteps": edges_step * args.steps / (total_ms / 1e3) / 1e9,
        "step": ("one mgk_khop_count_device_schedule call: group (300 seeds: k=1,2) = one on-chip k=2 launch whose "
                 "|F1| gives the k=1 answers; group (10 seeds: k=3,6) = one LANES traversal to depth 6 answering "
                 "both sections from its per-hop lane counts" if name == "cfg4" else "one schedule call"),
        "groups": groups,
        "roofline": {"bound": "hbm", "kernel": dom["kernel"] + f" (group k={dom['ks']})",
                     "achieved": dom["achieved_GBps"], "peak": pk["hbm_gbs"], "unit": "GB/s",
                     "frac": dom["frac_of_peak"], "peak_source": pk_src,
                     "algo_bytes_per_launch": dom["algo_bytes"],
                     "byte_model": "SURVEY.md §8(d): single-source 4E + 12 sum|F_l<L| + 4 sum|F_1..L|; "
                                   "64-lane mode 4 sum_U outdeg + 12|U| + 24 W n per level",
                     "traffic": (tr or {}).get("total") if tr else None,
                     "traffic_source": (tr or {}).get("source") if tr else "no ncu capture of this kernel on this workload"},
        "cpu_baseline": cpu,
        "parity": parity,
        "e2e": {"value": q_per_step * args.steps / (e2e_total / 1e3), "unit": "queries/s",
                "h2d_bytes_per_step": 4 * len(arm.seeds), "d2h_bytes_per_step": 8 * sum(arm.ns),
                "api": "k_hop_count_schedule (mgk_khop_count_schedule): host uint64 seeds in, host counts out",
                "ms_per_step": e2e_total / args.steps},
        "gpu_launches": sum(g["launches"] for g in groups) * args.steps,
        "clocks": clocks,
        "extra_configs": extras,
    }
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


# ---- the reference arm ---------------------------------------------------------------------
def run_reference(args):
    rank, _, world = dist_env()
    if rank != 0:
        return
    import oracle
    name = args.workload
    spec, ks, ns = SCHEDULE[name]
    cores = os.cpu_count() or 1
    P, R = oracle.Port(), oracle.Ref()
    t = time.time()
    rp, ci = P.gen_bench_csr(spec["scale"], spec["edge_factor"], spec["target_unique"], spec["relabel"])
    gen_s = time.time() - t
    n = len(rp) - 1
    m = len(ci)
    seeds = P.pick_seeds_u32(rp, SEEDS_PER_RANK, 1)
    t = time.time()
    M = R.matrix(rp, ci)
    prep_s = time.time() - t
    log(f"reference arm: {spec['name']} n={n} m={m} (oracle generator {gen_s:.0f}s, from_parts {prep_s:.0f}s)")
    del rp, ci
    # one step = the whole schedule as one job pool on all host threads (deep
    # queries first; each query on one thread, like the reference server)
    jobs_s, jobs_k = [], []
    for k, nn in sorted(zip(ks, ns), key=lambda x: -x[0]):
        jobs_s += [int(s) for s in seeds[:nn]]
        jobs_k += [k] * nn
    jobs_s = np.array(jobs_s, np.uint64)
    jobs_k = np.array(jobs_k, np.uint32)
    # warm-up: the k <= 2 part of the schedule (cheap), W times
    shallow = jobs_k <= 2
    for _ in range(args.warmup):
        M.khop_jobs(jobs_s[shallow], jobs_k[shallow], 0, threads=cores)
    budget = float(os.environ.get("MGK_REF_BUDGET_S", "150"))
    times, spent = [], 0.0
    while len(times) < args.steps and (not times or spent + times[-1] <= budget):
        _, el = M.khop_jobs(jobs_s, jobs_k, 0, threads=cores)
        times.append(el)
        spent += el
    total = float(np.sum(times))
    value = len(jobs_s) * len(times) / total
    line = {
        "metric": METRIC if name == "cfg4" else f"k-hop count queries/s ({name})",
        "value": value, "unit": "queries/s", "n_gpus": world, "steps": len(times), "steps_requested": args.steps,
        "warmup": args.warmup, "ms_per_step": total * 1e3 / len(times), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u64 vertex ids (integer)",
        "data": "synthetic R-MAT, BASELINE.json configs shape (seeded; stands in for the paper's Twitter / Graph500 graphs)",
        "config": workload_config(name, world, n, m),
        "impl": "reference",
        "cpu_baseline": {"value": value, "unit": "queries/s", "cores": cores, "kind": "reference",
                         "sample": f"{len(times)} step(s) of the full schedule ({len(jobs_s)} queries) on oracle/_ref "
                                   f"(unmodified matgraph core, -O3, checks off; matrix route: vxm/ewise_union loop "
                                   f"of execute.cpp:347-375 over from_parts), {cores} threads, one query per thread; "
                                   f"steps capped by a {budget:.0f}s budget"},
        "e2e": {"value": value, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "prep": {"oracle_generator_s": gen_s, "from_parts_s": prep_s},
        # evidence for the driver: this arm ran without the product library
        "product_library_loaded": product_library_loaded(),
    }
    print(json.dumps(line), flush=True)


def product_library_loaded() -> bool:
    try:
        with open("/proc/self/maps") as f:
            return any("libmgk" in ln or "libmatgraph_b200" in ln for ln in f)
    except OSError:
        return False


def relaunch_under_torchrun(args) -> int:
    """`python bench.py --gpus N` (N > 1) outside torchrun: re-launch this script
    with one process per GPU (rendezvous on 127.0.0.1)."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve())] + sys.argv[1:]
    log("relaunching under torchrun:", " ".join(cmd))
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg4", choices=sorted(SCHEDULE))
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-extras", action="store_true", help="skip the cfg2 / cfg3 / cfg5 sections")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world = int(os.environ.get("WORLD_SIZE", "0") or 0)
    if world == 0 and args.gpus > 1:
        sys.exit(relaunch_under_torchrun(args))
    if world and world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

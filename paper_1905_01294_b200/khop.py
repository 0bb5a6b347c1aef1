"""The k-hop count path, mirroring the reference's interface.

Reference (proj/core/include/matgraph/execute.hpp:52-68, execute.cpp:347-375):

    struct KHopQuery { uint64 seed; uint32 k = 1; RelationRef relation = ANY;
                       TraverseMode mode = Exact; };
    BitVector     k_hop_frontier(const PropertyGraph&, const KHopQuery&);
    std::uint64_t k_hop_count   (const PropertyGraph&, const KHopQuery&);

Here the graph argument is a :class:`DeviceGraph` — the device-resident
uint32 CSR + CSC of one relation matrix (what ``relation_matrix(rel)``
returns in the reference, proj/core/src/graph.cpp:84-88) — and the work runs
in the sm_100a kernels of libmgk.so through the C ABI. Errors mirror the
reference's classes and texts (proj/core/include/matgraph/error.hpp:10-66):
``ContractError("k-hop seed 99 is not an allocated node")`` etc.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import ENGINE_AUTO, ENGINE_LANES, ENGINE_SINGLE, MgkStats, MgkTuning

K_MAX_HOPS = 32  # proj/core/include/matgraph/ast.hpp:15


class Error(RuntimeError):
    """matgraph::Error (error.hpp:10-14)."""


class ContractError(Error):
    """matgraph::ContractError (error.hpp:16-19)."""


class HarnessError(Error):
    """matgraph::HarnessError (error.hpp:62-65)."""


class DeviceError(Error):
    """A CUDA failure inside the engine (reported as matgraph::Error)."""


class SnapshotError(Error):
    """matgraph::SnapshotError (error.hpp:52-61): malformed GRAPHSNAP1 text."""


def _raise(rc: int):
    msg = _lib.last_error()
    if rc == _lib.MGK_ECONTRACT:
        raise ContractError(msg)
    if rc == _lib.MGK_EHARNESS:
        raise HarnessError(msg)
    if rc == _lib.MGK_ERANGE:
        raise ContractError(msg)
    if rc == _lib.MGK_ESNAPSHOT:
        raise SnapshotError(msg)
    raise DeviceError(msg)


def _check(rc: int):
    if rc != _lib.MGK_OK:
        _raise(rc)


class TraverseMode(enum.IntEnum):
    """proj/core/include/matgraph/plan.hpp:17."""
    Exact = 0
    Cumulative = 1


@dataclass
class KHopQuery:
    """proj/core/include/matgraph/execute.hpp:53-58 (relation is chosen when the
    DeviceGraph is built, as relation_matrix(rel) is in the reference)."""
    seed: int = 0
    k: int = 1
    mode: TraverseMode = TraverseMode.Exact


@dataclass
class Tuning:
    alpha: int = 4
    beta: int = 24
    force_dir: int = 0   # 0 auto, 1 push only, 2 pull only
    lanes_words: int = 0  # 0 auto; else 1, 2, 4, 8 (x64 seeds per batch)
    alpha_lanes: int = 2
    alpha_last: int = 1


class DeviceGraph:
    """A relation matrix resident on one GPU (uint32 CSR + CSC + zero-in-degree bitmap)."""

    def __init__(self, handle: int, node_count: int | None = None):
        self._h = C.c_void_p(handle)
        n, m, dev = C.c_uint64(), C.c_uint64(), C.c_int()
        _check(_lib.lib().mgk_graph_info(self._h, C.byref(n), C.byref(m), C.byref(dev)))
        self.nrows, self.nnz, self.device = n.value, m.value, dev.value
        # KHopQuery seeds are checked against node_count (execute.cpp:348); the
        # store's capacity (matrix dimension) can be larger (graph.cpp:26).
        self.node_count = self.nrows if node_count is None else int(node_count)

    # -- construction ---------------------------------------------------------
    @classmethod
    def from_csr(cls, row_ptr, col_idx, device: int = 0, node_count: int | None = None):
        """Upload a SparseMatrix-shaped CSR (uint64 like the reference, or uint32)."""
        row_ptr = np.ascontiguousarray(row_ptr)
        col_idx = np.ascontiguousarray(col_idx)
        nrows = len(row_ptr) - 1
        h = C.c_void_p()
        L = _lib.lib()
        if row_ptr.dtype == np.uint32 and col_idx.dtype == np.uint32:
            ci = col_idx if len(col_idx) else np.zeros(1, np.uint32)
            _check(L.mgk_graph_upload_u32(device, nrows, len(col_idx), row_ptr.ctypes.data,
                                          ci.ctypes.data, C.byref(h)))
        else:
            rp = np.ascontiguousarray(row_ptr, np.uint64)
            ci = np.ascontiguousarray(col_idx, np.uint64)
            ci = ci if len(ci) else np.zeros(1, np.uint64)
            _check(L.mgk_graph_upload(device, nrows, len(col_idx), rp.ctypes.data, ci.ctypes.data,
                                      C.byref(h)))
        return cls(h.value, node_count)

    @classmethod
    def from_edges(cls, src, dst, node_count: int, device: int = 0):
        """build_bench_graph (bench.cpp:185-198) on the device: sort + dedup + CSR/CSC."""
        src = np.ascontiguousarray(src, np.uint32)
        dst = np.ascontiguousarray(dst, np.uint32)
        h = C.c_void_p()
        s = src if len(src) else np.zeros(1, np.uint32)
        d = dst if len(dst) else np.zeros(1, np.uint32)
        _check(_lib.lib().mgk_graph_from_edges(device, max(node_count, 1), len(src), s.ctypes.data,
                                               d.ctypes.data, C.byref(h)))
        return cls(h.value, node_count)

    @classmethod
    def generate(cls, spec, device: int = 0):
        """A harness.GraphSpec bench graph generated on the device (same graph
        as harness.gen_csr(spec), built with sort/dedup/CSR/CSC on the GPU)."""
        h = C.c_void_p()
        _check(_lib.lib().mgk_graph_gen_rmat(device, spec.scale, spec.edge_factor, spec.a, spec.b, spec.c,
                                             spec.rng_seed, spec.target_unique, spec.relabel, C.byref(h)))
        return cls(h.value)

    @classmethod
    def from_snapshot(cls, text=None, path=None, relation: str | None = None, device: int = 0):
        """GRAPHSNAP1 text (bytes) or file -> the device matrix of `relation`
        (None = ANY), parsed on the GPU (snapshot.cpp:162-259 + relation_matrix).
        node_count = the snapshot's NODES; malformed input raises SnapshotError
        with the reference's message."""
        h = C.c_void_p()
        n = C.c_uint64()
        rel = relation.encode() if relation is not None else None
        if path is not None:
            _check(_lib.lib().mgk_graph_load_snapshot_file(device, str(path).encode(), rel, C.byref(h), C.byref(n)))
        else:
            text = bytes(text)
            _check(_lib.lib().mgk_graph_load_snapshot(device, text, len(text), rel, C.byref(h), C.byref(n)))
        return cls(h.value, n.value)

    def replicate(self, device: int):
        """A copy of this device graph on `device` (peer copy over NVLink when
        it is another GPU): load-time replication for k_hop_count_multi."""
        h = C.c_void_p()
        _check(_lib.lib().mgk_graph_replicate(self.handle, device, C.byref(h)))
        return DeviceGraph(h.value, self.node_count)

    def transpose(self):
        """A^T as its own device graph (mgk_graph_transpose): traversals over it
        follow edges backwards (the `<-` direction of a Cypher pattern)."""
        h = C.c_void_p()
        _check(_lib.lib().mgk_graph_transpose(self.handle, C.byref(h)))
        return DeviceGraph(h.value, node_count=self.node_count)

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            _lib.lib().mgk_graph_free(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    # -- inspection -------------------------------------------------------------
    def csr(self):
        rp = np.zeros(self.nrows + 1, np.uint32)
        ci = np.zeros(max(self.nnz, 1), np.uint32)
        _check(_lib.lib().mgk_graph_download_csr(self._h, rp.ctypes.data, ci.ctypes.data))
        return rp, ci[: self.nnz]

    def csc(self):
        cp = np.zeros(self.nrows + 1, np.uint32)
        ri = np.zeros(max(self.nnz, 1), np.uint32)
        _check(_lib.lib().mgk_graph_download_csc(self._h, cp.ctypes.data, ri.ctypes.data))
        return cp, ri[: self.nnz]

    def device_bytes(self) -> int:
        return int(_lib.lib().mgk_graph_device_bytes(self._h))

    def set_tuning(self, t: Tuning):
        tt = MgkTuning(t.alpha, t.beta, t.force_dir, t.lanes_words, t.alpha_lanes, t.alpha_last)
        _check(_lib.lib().mgk_graph_set_tuning(self._h, C.byref(tt)))

    def get_tuning(self) -> Tuning:
        tt = MgkTuning()
        _check(_lib.lib().mgk_graph_get_tuning(self._h, C.byref(tt)))
        return Tuning(tt.alpha, tt.beta, tt.force_dir, tt.lanes_words, tt.alpha_lanes, tt.alpha_last)

    def _check_seed(self, seed: int):
        if seed < 0 or seed >= self.node_count:
            raise ContractError(f"k-hop seed {seed} is not an allocated node")


def _check_k(k: int):
    if k < 1 or k > K_MAX_HOPS:
        raise ContractError(f"k-hop count {k} outside [1, {K_MAX_HOPS}]")


def k_hop_count(graph: DeviceGraph, query: KHopQuery) -> int:
    """execute.cpp:373-375 — number of vertices in k_hop_frontier(graph, query)."""
    graph._check_seed(query.seed)
    _check_k(query.k)
    return int(k_hop_count_batch(graph, [query.seed], query.k, query.mode)[0])


def k_hop_frontier(graph: DeviceGraph, query: KHopQuery) -> np.ndarray:
    """execute.cpp:347-371 — sorted uint64 ids (exact: distance == k; cumulative: 1..k)."""
    graph._check_seed(query.seed)
    _check_k(query.k)
    cap = max(graph.nrows, 1)
    ids = np.zeros(cap, np.uint64)
    n = C.c_uint64()
    _check(_lib.lib().mgk_khop_frontier(graph.handle, int(query.seed), int(query.k),
                                        int(query.mode), ids.ctypes.data, cap, C.byref(n)))
    return ids[: n.value].copy()


def k_hop_count_batch(graph: DeviceGraph, seeds, k: int, mode=TraverseMode.Exact,
                      engine: int = ENGINE_AUTO, stats: bool = False):
    """Batched k_hop_count: one count per seed, host buffers (additive API).

    Seeds are validated in order exactly like k_hop_frontier's first check.
    With stats=True returns (counts, stats_dict) with per-hop work counters.
    """
    seeds = np.ascontiguousarray(seeds, np.uint64)
    if graph.node_count < graph.nrows and len(seeds):  # the C ABI checks against nrows
        bad = np.flatnonzero(seeds >= graph.node_count)
        if len(bad):
            raise ContractError(f"k-hop seed {int(seeds[bad[0]])} is not an allocated node")
    _check_k(k)
    counts = np.empty(max(len(seeds), 1), np.uint64)
    st = MgkStats() if stats else None
    sp = seeds if len(seeds) else np.zeros(1, np.uint64)
    _check(_lib.lib().mgk_khop_count_ex(graph.handle, sp.ctypes.data, len(seeds), int(k), int(mode),
                                        int(engine), counts.ctypes.data,
                                        C.byref(st) if stats else None))
    counts = counts[: len(seeds)]
    return (counts, st.to_dict()) if stats else counts


def walk_count_batch(graph: DeviceGraph, sources, min_hops: int, max_hops: int,
                     engine: int = ENGINE_AUTO):
    """|walk_targets(src, min, max)| per source (execute.cpp:43-60): the
    VarLenTraverse step of MATCH (a)-[*min..max]->(b) — visited starts empty,
    so the source itself is counted when a cycle returns to it."""
    src = np.ascontiguousarray(sources, np.uint64)
    counts = np.zeros(max(len(src), 1), np.uint64)
    sp = src if len(src) else np.zeros(1, np.uint64)
    _check(_lib.lib().mgk_walk_count(graph.handle, sp.ctypes.data, len(src), int(min_hops), int(max_hops),
                                     int(engine), counts.ctypes.data))
    return counts[: len(src)]


def walk_targets(graph: DeviceGraph, source: int, min_hops: int, max_hops: int) -> np.ndarray:
    """execute.cpp:43-60 walk_targets: sorted ids of walk levels min..max."""
    cap = max(graph.nrows, 1)
    ids = np.zeros(cap, np.uint64)
    n = C.c_uint64()
    _check(_lib.lib().mgk_walk_targets(graph.handle, int(source), int(min_hops), int(max_hops),
                                       ids.ctypes.data, cap, C.byref(n)))
    return ids[: n.value].copy()


SEMIRING_BOOL_OR_AND, SEMIRING_PLUS_TIMES, SEMIRING_MIN_PLUS = 0, 1, 2  # sparse.hpp:54-66


def mxm(a, b, semiring: int = SEMIRING_BOOL_OR_AND, mask=None, device: int = 0):
    """mxm (sparse.cpp:292-363) on the GPU. Matrices are (nrows, ncols,
    row_ptr, col_idx, vals|None) host tuples (vals None = structural);
    returns the same shape (vals None for a structural / empty result)."""
    def args(m):
        nr, nc, rp, ci, v = m
        rp = np.ascontiguousarray(rp, np.uint64)
        ci = np.ascontiguousarray(ci, np.uint64) if len(ci) else np.zeros(1, np.uint64)
        v = None if v is None else (np.ascontiguousarray(v, np.int64) if len(v) else np.zeros(1, np.int64))
        return int(nr), int(nc), rp, ci, v
    an, ac, arp, aci, av = args(a)
    bn, bc, brp, bci, bv = args(b)
    mn = mc = 0
    mrp = mci = None
    if mask is not None:
        mn, mc, mrp, mci, _ = args(mask)
    ptr = lambda x: None if x is None else x.ctypes.data  # noqa: E731
    h = C.c_void_p()
    _check(_lib.lib().mgk_mxm(device, an, ac, ptr(arp), ptr(aci), ptr(av), bn, bc, ptr(brp), ptr(bci), ptr(bv),
                              int(semiring), mn, mc, ptr(mrp), ptr(mci), C.byref(h)))
    try:
        nr, nc, nnz, valued = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_int()
        _check(_lib.lib().mgk_matrix_info(h, C.byref(nr), C.byref(nc), C.byref(nnz), C.byref(valued)))
        rp = np.empty(nr.value + 1, np.uint64)
        ci = np.empty(nnz.value, np.uint64)
        vals = np.empty(nnz.value, np.int64) if valued.value else None
        _check(_lib.lib().mgk_matrix_download(h, rp.ctypes.data, ci.ctypes.data if nnz.value else None,
                                              vals.ctypes.data if vals is not None and nnz.value else None))
    finally:
        _lib.lib().mgk_matrix_free(h)
    return nr.value, nc.value, rp, ci, vals


def snapshot_check(text: bytes):
    """The GRAPHSNAP1 grammar on the host only (no GPU): (NODES, EDGES) or SnapshotError."""
    text = bytes(text)
    n, m = C.c_uint64(), C.c_uint64()
    _check(_lib.lib().mgk_snapshot_check(text, len(text), C.byref(n), C.byref(m)))
    return n.value, m.value


def k_hop_count_sections(graph: DeviceGraph, seeds, ks, mode=TraverseMode.Exact):
    """k_hop_count for every seed at every k in `ks`, one call (the
    harness's sections over one master seed list, bench.cpp:311-343):
    returns uint64 counts of shape (len(ks), len(seeds))."""
    seeds = np.ascontiguousarray(seeds, np.uint64)
    ks = np.ascontiguousarray(ks, np.uint32)
    if graph.node_count < graph.nrows and len(seeds):  # the C ABI checks against nrows
        bad = np.flatnonzero(seeds >= graph.node_count)
        if len(bad):
            raise ContractError(f"k-hop seed {int(seeds[bad[0]])} is not an allocated node")
    for k in ks:
        _check_k(int(k))
    counts = np.empty((len(ks), len(seeds)), np.uint64)
    if len(ks) and len(seeds):
        _check(_lib.lib().mgk_khop_count_ks(graph.handle, seeds.ctypes.data, len(seeds), ks.ctypes.data, len(ks),
                                            int(mode), counts.ctypes.data))
    return counts


def k_hop_count_schedule(graph: DeviceGraph, seeds, nseeds_per_k, ks, mode=TraverseMode.Exact):
    """The harness's whole schedule in one call (run_khop_benchmark,
    bench.cpp:311-343): section j = k_hop_count(seeds[i], ks[j]) for the
    prefix i < nseeds_per_k[j] of one master list. Returns a list of uint64
    arrays, one per section (mgk_khop_count_schedule)."""
    seeds = np.ascontiguousarray(seeds, np.uint64)
    ns = np.ascontiguousarray(nseeds_per_k, np.uint64)
    ks = np.ascontiguousarray(ks, np.uint32)
    if len(ns) != len(ks):
        raise ContractError(f"schedule pairs {len(ks)} hop counts with {len(ns)} seed counts")
    if len(ns) and int(ns.max()) > len(seeds):
        raise ContractError(f"schedule needs {int(ns.max())} seeds, {len(seeds)} given")
    if graph.node_count < graph.nrows and len(seeds) and len(ns):  # the C ABI checks against nrows
        bad = np.flatnonzero(seeds[: int(ns.max())] >= graph.node_count)
        if len(bad):
            raise ContractError(f"k-hop seed {int(seeds[bad[0]])} is not an allocated node")
    counts = np.zeros(max(int(ns.sum()) if len(ns) else 0, 1), np.uint64)
    if len(ks):
        _check(_lib.lib().mgk_khop_count_schedule(graph.handle, seeds.ctypes.data if len(seeds) else None,
                                                  ns.ctypes.data, ks.ctypes.data, len(ks), int(mode),
                                                  counts.ctypes.data))
    out, off = [], 0
    for n in ns.tolist():
        out.append(counts[off:off + n].copy())
        off += n
    return out


def k_hop_count_device_schedule(graph: DeviceGraph, d_seeds_ptr: int, nseeds_per_k, ks, mode: int,
                                d_counts_ptr: int, stream_ptr: int = 0):
    """Device-resident schedule (mgk_khop_count_device_schedule): sections back
    to back in d_counts (uint64), async on the stream."""
    ns = np.ascontiguousarray(nseeds_per_k, np.uint64)
    ks = np.ascontiguousarray(ks, np.uint32)
    _check(_lib.lib().mgk_khop_count_device_schedule(graph.handle, C.c_void_p(d_seeds_ptr), ns.ctypes.data,
                                                     ks.ctypes.data, len(ks), int(mode), C.c_void_p(d_counts_ptr),
                                                     C.c_void_p(stream_ptr)))


def k_hop_count_multi(replicas, seeds, k: int, mode=TraverseMode.Exact):
    """One batch over replicas of the same graph (e.g. one per GPU, made with
    DeviceGraph.replicate): contiguous seed shards, one host thread per
    replica, no collective. Same answers and errors as
    k_hop_count_batch."""
    reps = list(replicas)
    if not reps:
        raise ContractError("no replicas")
    seeds = np.ascontiguousarray(seeds, np.uint64)
    node_count = reps[0].node_count
    if node_count < reps[0].nrows and len(seeds):
        bad = np.flatnonzero(seeds >= node_count)
        if len(bad):
            raise ContractError(f"k-hop seed {int(seeds[bad[0]])} is not an allocated node")
    _check_k(k)
    counts = np.empty(max(len(seeds), 1), np.uint64)
    handles = (C.c_void_p * len(reps))(*[r.handle for r in reps])
    sp = seeds if len(seeds) else np.zeros(1, np.uint64)
    _check(_lib.lib().mgk_khop_count_multi(handles, len(reps), sp.ctypes.data, len(seeds), int(k), int(mode),
                                           counts.ctypes.data))
    return counts[: len(seeds)]


def k_hop_count_device(graph: DeviceGraph, d_seeds_ptr: int, nseeds: int, k: int, mode: int,
                       d_counts_ptr: int, stream_ptr: int = 0, engine: int = ENGINE_AUTO):
    """Device-resident batch: uint32 seeds and uint64 counts already in HBM; async on stream."""
    _check(_lib.lib().mgk_khop_count_device(graph.handle, C.c_void_p(d_seeds_ptr), nseeds, int(k),
                                            int(mode), int(engine), C.c_void_p(d_counts_ptr),
                                            C.c_void_p(stream_ptr)))


def k_hop_count_device_sections(graph: DeviceGraph, d_seeds_ptr: int, nseeds: int, ks, mode: int,
                                d_counts_ptr: int, stream_ptr: int = 0):
    """Device-resident sections: the answers for ks[j] at d_counts[j * nseeds + i]
    (uint64), async on stream. A k = 1 section rides on the on-chip k = 2 launch."""
    ks = np.ascontiguousarray(ks, np.uint32)
    _check(_lib.lib().mgk_khop_count_device_ks(graph.handle, C.c_void_p(d_seeds_ptr), nseeds, ks.ctypes.data,
                                               len(ks), int(mode), C.c_void_p(d_counts_ptr),
                                               C.c_void_p(stream_ptr)))


def device_check(graph: DeviceGraph, stream_ptr: int = 0) -> None:
    """mgk_khop_device_check: wait for the stream; ContractError when a
    device-path call met a seed >= node count since the last check."""
    _check(_lib.lib().mgk_khop_device_check(graph.handle, C.c_void_p(stream_ptr)))


def device_stats(graph: DeviceGraph, stream_ptr: int = 0) -> dict:
    st = MgkStats()
    _check(_lib.lib().mgk_khop_device_stats(graph.handle, C.c_void_p(stream_ptr), C.byref(st)))
    return st.to_dict()


def device_count() -> int:
    return int(_lib.lib().mgk_device_count())


__all__ = ["ContractError", "HarnessError", "Error", "DeviceError", "SnapshotError", "snapshot_check", "mxm",
           "SEMIRING_BOOL_OR_AND", "SEMIRING_PLUS_TIMES", "SEMIRING_MIN_PLUS", "TraverseMode", "KHopQuery",
           "Tuning", "DeviceGraph", "k_hop_count", "k_hop_frontier", "k_hop_count_batch",
           "k_hop_count_device", "k_hop_count_device_sections", "k_hop_count_schedule",
           "k_hop_count_device_schedule", "k_hop_count_multi", "k_hop_count_sections", "walk_count_batch",
           "walk_targets", "device_stats", "device_check", "device_count", "ENGINE_AUTO", "ENGINE_SINGLE",
           "ENGINE_LANES", "K_MAX_HOPS"]

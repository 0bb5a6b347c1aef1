"""TEST INFRASTRUCTURE ONLY — ctypes bindings for the k-hop CPU oracle.

Two checkers live here (see oracle/Makefile):

* ``Port``  — ``liboracle.so``, the plain-C restatement of the reference
  algorithm (oracle/khop_oracle.c, each function citing the reference
  file:line it follows).
* ``Ref``   — ``_ref/libmatgraph_ref.so``, the unmodified reference core
  (/root/reference/proj/core/src) compiled in place with its namespace renamed
  to ``matgraph_ref`` plus the thin C wrapper oracle/ref_capi.cpp.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this module, and only
as the checker / CPU baseline. The product package
``paper_1905_01294_b200`` never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
PORT_SO = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / "libmatgraph_ref.so"

EXACT, CUMULATIVE = 0, 1
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")


def build(ref: bool | None = None) -> None:
    """Build liboracle.so (always) and the reference .so (when /root/reference exists)."""
    import subprocess

    targets = ["oracle"]
    if ref or (ref is None and Path("/root/reference/proj/core/src").is_dir()):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", str(HERE), f"-j{os.cpu_count() or 4}", *targets], check=True)


class Port:
    """The plain-C restatement (oracle/khop_oracle.c)."""

    def __init__(self, path: Path = PORT_SO):
        if not path.exists():
            build(ref=False)
        L = self.lib = C.CDLL(str(path))
        L.orc_rmat_generate.restype = C.c_uint64
        L.orc_rmat_generate.argtypes = [C.c_uint32, C.c_uint32, C.c_double, C.c_double, C.c_double,
                                        C.c_uint64, C.c_void_p, C.c_void_p]
        L.orc_build_csr.restype = C.c_uint64
        L.orc_build_csr.argtypes = [C.c_uint64, C.c_uint64, _u32p, _u32p, _u64p, _u64p]
        L.orc_pick_seeds.restype = C.c_int
        L.orc_pick_seeds.argtypes = [C.c_uint64, _u64p, C.c_uint64, C.c_uint64, _u64p,
                                     C.POINTER(C.c_uint64)]
        L.orc_adj_new.restype = C.c_void_p
        L.orc_adj_new.argtypes = [C.c_uint64, C.c_uint64, _u32p, _u32p]
        L.orc_adj_free.argtypes = [C.c_void_p]
        L.orc_bfs_count.restype = C.c_uint64
        L.orc_bfs_count.argtypes = [C.c_void_p, C.c_uint64, C.c_uint32, C.c_int]
        L.orc_khop_frontier.restype = C.c_uint64
        L.orc_khop_frontier.argtypes = [C.c_uint64, _u64p, _u64p, C.c_uint64, C.c_uint32, C.c_int,
                                        C.c_void_p]
        L.orc_walk_targets.restype = C.c_uint64
        L.orc_walk_targets.argtypes = [C.c_uint64, _u64p, _u64p, C.c_uint64, C.c_uint32, C.c_uint32,
                                       C.c_void_p]
        vp = C.c_void_p
        L.orc_mxm.restype = C.c_uint64
        L.orc_mxm.argtypes = [C.c_uint64, vp, vp, vp, C.c_uint64, vp, vp, vp, C.c_int, vp, vp, vp, vp, vp]
        L.orc_khop_work.restype = C.c_uint64
        L.orc_khop_work.argtypes = [C.c_uint64, _u64p, _u64p, C.c_uint64, C.c_uint32, C.c_void_p,
                                    C.POINTER(C.c_uint32)]

        L.orc_gen_bench_csr.restype = C.c_int
        L.orc_gen_bench_csr.argtypes = [C.c_uint32, C.c_uint32, C.c_double, C.c_double, C.c_double, C.c_uint64,
                                        C.c_uint64, C.c_int, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                        C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)]
        L.orc_free.argtypes = [C.c_void_p]
        L.orc_set_threads.argtypes = [C.c_uint]
        L.orc_pick_seeds_u32.restype = C.c_int
        L.orc_pick_seeds_u32.argtypes = [C.c_uint64, _u32p, C.c_uint64, C.c_uint64, _u64p, C.POINTER(C.c_uint64)]
        L.orc_khop_many.restype = None
        L.orc_khop_many.argtypes = [C.c_uint64, _u32p, _u32p, _u64p, C.c_uint64, C.c_uint32, C.c_uint,
                                    C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]

    def rmat_generate(self, scale, edge_factor=16, a=0.57, b=0.19, c=0.19, rng_seed=1):
        m = self.lib.orc_rmat_generate(scale, edge_factor, a, b, c, rng_seed, None, None)
        src = np.empty(m, np.uint32)
        dst = np.empty(m, np.uint32)
        self.lib.orc_rmat_generate(scale, edge_factor, a, b, c, rng_seed,
                                   src.ctypes.data, dst.ctypes.data)
        return src, dst

    def build_csr(self, n, src, dst):
        src = np.ascontiguousarray(src, np.uint32)
        dst = np.ascontiguousarray(dst, np.uint32)
        row_ptr = np.zeros(n + 1, np.uint64)
        col_idx = np.zeros(max(len(src), 1), np.uint64)
        nnz = self.lib.orc_build_csr(n, len(src), src, dst, row_ptr, col_idx)
        if nnz == (1 << 64) - 1:
            raise ValueError("edge endpoint outside the node range")
        return row_ptr, col_idx[:nnz].copy()

    def pick_seeds(self, row_ptr, n, rng_seed):
        node_count = len(row_ptr) - 1
        out = np.zeros(max(n, 1), np.uint64)
        elig = C.c_uint64(0)
        rc = self.lib.orc_pick_seeds(node_count, np.ascontiguousarray(row_ptr, np.uint64), n,
                                     rng_seed, out, C.byref(elig))
        if rc != 0:
            raise RuntimeError(f"need {n} seeds but only {elig.value} nodes have out-degree >= 1")
        return out[:n].copy()

    def bfs_oracle(self, n, src, dst):
        return _Adj(self.lib, n, src, dst)

    def khop_frontier(self, row_ptr, col_idx, seed, k, mode):
        n = len(row_ptr) - 1
        out = np.zeros(max(n, 1), np.uint64)
        cnt = self.lib.orc_khop_frontier(n, row_ptr, _c64(col_idx), seed, k, mode, out.ctypes.data)
        return out[:cnt].copy()

    def khop_count(self, row_ptr, col_idx, seed, k, mode):
        n = len(row_ptr) - 1
        return int(self.lib.orc_khop_frontier(n, row_ptr, _c64(col_idx), seed, k, mode, None))

    def walk_targets(self, row_ptr, col_idx, src, lo, hi):
        """execute.cpp:43-60: sorted union of walk levels lo..hi (nothing pre-visited)."""
        n = len(row_ptr) - 1
        out = np.zeros(max(n, 1), np.uint64)
        cnt = self.lib.orc_walk_targets(n, row_ptr, _c64(col_idx), src, lo, hi, out.ctypes.data)
        return out[:cnt].copy()

    def khop_work(self, row_ptr, col_idx, seed, k):
        """(E(s,k), level sizes [|F_0|..|F_L|]) — SURVEY.md §8(d)."""
        n = len(row_ptr) - 1
        sizes = np.zeros(k + 1, np.uint64)
        L = C.c_uint32(0)
        e = self.lib.orc_khop_work(n, row_ptr, _c64(col_idx), seed, k, sizes.ctypes.data, C.byref(L))
        return int(e), sizes[: L.value + 1].copy()


    # ---- bench scale (oracle/bench_oracle.c) ---------------------------------
    def gen_bench_csr(self, scale, edge_factor=16, target_unique=0, relabel=1, a=0.57, b=0.19, c=0.19,
                      rng_seed=1):
        """The BASELINE.json bench graph as a uint32 CSR (row_ptr, col_idx):
        the chunked R-MAT stream's first `target_unique` distinct non-loop
        edges, relabelled (bench_oracle.c orc_gen_bench_csr)."""
        n, m = C.c_uint64(), C.c_uint64()
        prp, pci = C.c_void_p(), C.c_void_p()
        rc = self.lib.orc_gen_bench_csr(scale, edge_factor, a, b, c, rng_seed, target_unique, relabel,
                                        C.byref(n), C.byref(m), C.byref(prp), C.byref(pci))
        if rc != 0:
            raise MemoryError("orc_gen_bench_csr failed (allocation or uint32 range)")
        try:
            rp = np.ctypeslib.as_array(C.cast(prp, C.POINTER(C.c_uint32)), (n.value + 1,)).copy()
            ci = np.ctypeslib.as_array(C.cast(pci, C.POINTER(C.c_uint32)), (max(m.value, 1),))[: m.value].copy()
        finally:
            self.lib.orc_free(prp)
            self.lib.orc_free(pci)
        return rp, ci

    def gen_spec(self, spec):
        """gen_bench_csr for a harness GraphSpec-like object (name, scale, ...)."""
        return self.gen_bench_csr(spec.scale, spec.edge_factor, spec.target_unique, spec.relabel, spec.a,
                                  spec.b, spec.c, spec.rng_seed)

    def pick_seeds_u32(self, row_ptr, n, rng_seed):
        """bench.cpp:200-218 over a uint32 CSR."""
        rp = np.ascontiguousarray(row_ptr, np.uint32)
        out = np.zeros(max(n, 1), np.uint64)
        elig = C.c_uint64(0)
        if self.lib.orc_pick_seeds_u32(len(rp) - 1, rp, n, rng_seed, out, C.byref(elig)) != 0:
            raise RuntimeError(f"need {n} seeds but only {elig.value} nodes have out-degree >= 1")
        return out[:n].copy()

    def khop_many(self, row_ptr, col_idx, seeds, k, threads=0, work=False):
        """(exact[ns], cumulative[ns]) of k_hop_count for every seed on all host
        threads; with work=True also (E[ns], levels[ns, k+1])."""
        rp = np.ascontiguousarray(row_ptr, np.uint32)
        ci = np.ascontiguousarray(col_idx, np.uint32)
        if len(ci) == 0:
            ci = np.zeros(1, np.uint32)
        sd = np.ascontiguousarray(seeds, np.uint64)
        ns = len(sd)
        ex = np.zeros(max(ns, 1), np.uint64)
        cu = np.zeros(max(ns, 1), np.uint64)
        ed = np.zeros(max(ns, 1), np.uint64) if work else None
        lv = np.zeros((max(ns, 1), k + 1), np.uint64) if work else None
        if ns:
            self.lib.orc_khop_many(len(rp) - 1, rp, ci, sd, ns, k, threads, ex.ctypes.data, cu.ctypes.data,
                                   None if ed is None else ed.ctypes.data, None if lv is None else lv.ctypes.data)
        if work:
            return ex[:ns], cu[:ns], ed[:ns], lv[:ns]
        return ex[:ns], cu[:ns]

def _csr_args(m):
    """(nrows, ncols, row_ptr, col_idx, vals|None) -> contiguous arrays kept alive by the caller."""
    nr, nc, rp, ci, v = m
    rp = np.ascontiguousarray(rp, np.uint64)
    ci = _c64(ci)
    v = None if v is None else (np.ascontiguousarray(v, np.int64) if len(v) else np.zeros(1, np.int64))
    return int(nr), int(nc), rp, ci, v


def _ptr(a):
    return None if a is None else a.ctypes.data


def _port_mxm(self, a, b, semiring=0, mask=None):
    """sparse.cpp:292-363 restated (oracle/khop_oracle.c orc_mxm). Matrices are
    (nrows, ncols, row_ptr, col_idx, vals|None); returns the same tuple."""
    an, ac, arp, aci, av = _csr_args(a)
    bn, bc, brp, bci, bv = _csr_args(b)
    mrp = mci = None
    if mask is not None:
        _, _, mrp, mci, _ = _csr_args(mask)
    args = (an, _ptr(arp), _ptr(aci), _ptr(av), bc, _ptr(brp), _ptr(bci), _ptr(bv), semiring, _ptr(mrp), _ptr(mci))
    nnz = self.lib.orc_mxm(*args, None, None, None)
    rp = np.zeros(an + 1, np.uint64)
    ci = np.zeros(max(nnz, 1), np.uint64)
    vals = np.zeros(max(nnz, 1), np.int64)
    self.lib.orc_mxm(*args, rp.ctypes.data, ci.ctypes.data, vals.ctypes.data)
    return an, bc, rp, ci[:nnz].copy(), (vals[:nnz].copy() if semiring != 0 and nnz else None)


Port.mxm = _port_mxm


def _c64(a):
    a = np.ascontiguousarray(a, np.uint64)
    return a if len(a) else np.zeros(1, np.uint64)


class _Adj:
    def __init__(self, lib, n, src, dst):
        self.lib = lib
        self._src = np.ascontiguousarray(src, np.uint32)
        self._dst = np.ascontiguousarray(dst, np.uint32)
        self.h = lib.orc_adj_new(n, len(self._src), _nz32(self._src), _nz32(self._dst))

    def count(self, seed, k, mode):
        return int(self.lib.orc_bfs_count(self.h, seed, k, mode))

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.orc_adj_free(self.h)
            self.h = None


def _nz32(a):
    return a if len(a) else np.zeros(1, np.uint32)


class RefError(Exception):
    """An exception raised inside the reference (message = its what())."""

    def __init__(self, code: int, message: str):
        super().__init__(message)
        self.code = code  # 1 ContractError, 2 HarnessError, 3 other matgraph::Error


class Ref:
    """The unmodified reference core, via oracle/ref_capi.cpp."""

    def __init__(self, path: Path = REF_SO):
        if not path.exists():
            raise FileNotFoundError(f"{path} not built (run make -C oracle ref where /root/reference exists)")
        L = self.lib = C.CDLL(str(path))
        vp, u64, u32 = C.c_void_p, C.c_uint64, C.c_uint32
        L.ref_last_error.restype = C.c_char_p
        L.ref_graph_new.restype = vp
        L.ref_graph_new.argtypes = [u64]
        L.ref_graph_create_nodes.argtypes = [vp, u64]
        L.ref_graph_create_edge.argtypes = [vp, u64, C.c_char_p, u64]
        L.ref_build_bench_graph.argtypes = [vp, vp, u64, u64, C.POINTER(vp)]
        L.ref_graph_free.argtypes = [vp]
        L.ref_graph_node_count.restype = u64
        L.ref_graph_node_count.argtypes = [vp]
        L.ref_graph_relation_csr.argtypes = [vp, C.c_char_p, C.POINTER(u64), C.POINTER(u64), vp, vp]
        L.ref_k_hop_count.argtypes = [vp, u64, u32, C.c_int, C.c_char_p, C.POINTER(u64)]
        L.ref_k_hop_frontier.argtypes = [vp, u64, u32, C.c_int, C.c_char_p, vp, u64, C.POINTER(u64)]
        L.ref_k_hop_count_many.argtypes = [vp, vp, u64, u32, C.c_int, C.c_int, vp,
                                           C.POINTER(C.c_double)]
        L.ref_pick_seeds.argtypes = [vp, u64, u64, vp]
        L.ref_cypher.argtypes = [vp, C.c_char_p, C.c_char_p, u64, C.POINTER(u64)]
        L.ref_rmat_generate.argtypes = [u32, u32, C.c_double, C.c_double, C.c_double, C.c_double,
                                        u64, vp, vp, C.POINTER(u64)]
        L.ref_graph_create_node_full.argtypes = [vp, C.c_char_p, C.c_char_p]
        L.ref_graph_create_edge_props.argtypes = [vp, u64, C.c_char_p, u64, C.c_char_p]
        L.ref_snapshot_parse.argtypes = [C.c_char_p, u64, C.POINTER(vp)]
        L.ref_snapshot_to_string.argtypes = [vp, C.c_char_p, u64, C.POINTER(u64)]
        L.ref_mxm.argtypes = [u64, u64, vp, vp, vp, u64, u64, vp, vp, vp, C.c_int, u64, u64, vp, vp,
                              C.POINTER(u64), C.POINTER(C.c_int), vp, vp, vp]
        L.ref_bfs_oracle_new.restype = vp
        L.ref_bfs_oracle_new.argtypes = [vp, vp, u64, u64]
        L.ref_bfs_oracle_count.argtypes = [vp, u64, u32, C.c_int, C.POINTER(u64)]
        L.ref_bfs_oracle_free.argtypes = [vp]
        L.ref_matrix_from_csr_u32.restype = vp
        L.ref_matrix_from_csr_u32.argtypes = [u64, vp, vp]
        L.ref_matrix_free.argtypes = [vp]
        L.ref_matrix_khop_jobs.argtypes = [vp, vp, vp, u64, C.c_int, C.c_int, vp, C.POINTER(C.c_double)]
        L.ref_graph_khop_jobs.argtypes = [vp, vp, vp, u64, C.c_int, C.c_int, vp, C.POINTER(C.c_double)]

    def _check(self, rc):
        if rc != 0:
            raise RefError(rc, self.lib.ref_last_error().decode())

    # graphs
    def graph(self, capacity=16):
        return RefGraph(self, self.lib.ref_graph_new(capacity))

    def build_bench_graph(self, src, dst, node_count):
        src = np.ascontiguousarray(src, np.uint32)
        dst = np.ascontiguousarray(dst, np.uint32)
        h = C.c_void_p()
        self._check(self.lib.ref_build_bench_graph(src.ctypes.data, dst.ctypes.data, len(src),
                                                   node_count, C.byref(h)))
        return RefGraph(self, h.value)

    def mxm(self, a, b, semiring=0, mask=None):
        """The reference's mxm over from_parts operands; returns
        (nrows, ncols, row_ptr, col_idx, vals|None)."""
        an, ac, arp, aci, av = _csr_args(a)
        bn, bc, brp, bci, bv = _csr_args(b)
        mn = mc = 0
        mrp = mci = None
        if mask is not None:
            mn, mc, mrp, mci, _ = _csr_args(mask)
        nnz, valued = C.c_uint64(), C.c_int()
        args = (an, ac, _ptr(arp), _ptr(aci), _ptr(av), bn, bc, _ptr(brp), _ptr(bci), _ptr(bv), semiring,
                mn, mc, _ptr(mrp), _ptr(mci), C.byref(nnz), C.byref(valued))
        self._check(self.lib.ref_mxm(*args, None, None, None))
        rp = np.zeros(an + 1, np.uint64)
        ci = np.zeros(max(nnz.value, 1), np.uint64)
        vals = np.zeros(max(nnz.value, 1), np.int64)
        self._check(self.lib.ref_mxm(*args, rp.ctypes.data, ci.ctypes.data, vals.ctypes.data))
        n = nnz.value
        return an, bc, rp, ci[:n].copy(), (vals[:n].copy() if valued.value else None)

    def snapshot_parse(self, text: bytes):
        """snapshot_from_string (snapshot.cpp:162-231); raises RefError with its message."""
        h = C.c_void_p()
        self._check(self.lib.ref_snapshot_parse(text, len(text), C.byref(h)))
        return RefGraph(self, h.value)

    def rmat_generate(self, scale, edge_factor=16, a=0.57, b=0.19, c=0.19, d=0.05, rng_seed=1):
        m = C.c_uint64(0)
        self._check(self.lib.ref_rmat_generate(scale, edge_factor, a, b, c, d, rng_seed, None, None,
                                               C.byref(m)))
        src = np.empty(m.value, np.uint32)
        dst = np.empty(m.value, np.uint32)
        self._check(self.lib.ref_rmat_generate(scale, edge_factor, a, b, c, d, rng_seed,
                                               src.ctypes.data, dst.ctypes.data, C.byref(m)))
        return src, dst

    def matrix(self, row_ptr, col_idx):
        """The reference's SparseMatrix::from_parts over a uint32 CSR (validated by
        the reference); k_hop jobs then run the k_hop_frontier loop on it with
        the PropertyGraph wrapper bypassed (ref_capi.cpp)."""
        rp = np.ascontiguousarray(row_ptr, np.uint32)
        ci = np.ascontiguousarray(col_idx, np.uint32)
        if len(ci) == 0:
            ci = np.zeros(1, np.uint32)
        h = self.lib.ref_matrix_from_csr_u32(len(rp) - 1, rp.ctypes.data, ci.ctypes.data)
        if not h:
            raise RefError(3, self.lib.ref_last_error().decode())
        return RefMatrix(self, h)

    def bfs_oracle(self, src, dst, n):
        src = np.ascontiguousarray(src, np.uint32)
        dst = np.ascontiguousarray(dst, np.uint32)
        h = self.lib.ref_bfs_oracle_new(src.ctypes.data, dst.ctypes.data, len(src), n)
        if not h:
            raise RefError(1, self.lib.ref_last_error().decode())
        return RefBfs(self, h)


def _jobs(ref, fn, h, seeds, ks, mode, threads):
    seeds = np.ascontiguousarray(seeds, np.uint64)
    ks = np.ascontiguousarray(ks, np.uint32)
    counts = np.zeros(max(len(seeds), 1), np.uint64)
    el = C.c_double()
    ref._check(fn(h, seeds.ctypes.data, ks.ctypes.data, len(seeds), mode, threads, counts.ctypes.data,
                  C.byref(el)))
    return counts[: len(seeds)], el.value


class RefMatrix:
    """A bare reference SparseMatrix (the 'wrapper bypassed' route for G4)."""

    def __init__(self, ref: Ref, h):
        self.ref, self.h = ref, h

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.lib.ref_matrix_free(self.h)
            self.h = None

    def khop_jobs(self, seeds, ks, mode=EXACT, threads=1):
        """(counts, wall seconds) of jobs i = (seeds[i], ks[i]), one query per thread."""
        return _jobs(self.ref, self.ref.lib.ref_matrix_khop_jobs, self.h, seeds, ks, mode, threads)


class RefGraph:
    def __init__(self, ref: Ref, h):
        self.ref, self.h = ref, h

    def khop_jobs(self, seeds, ks, mode=EXACT, threads=1):
        """(counts, wall seconds) of k_hop_count(seeds[i], ks[i]) jobs, one query per thread."""
        return _jobs(self.ref, self.ref.lib.ref_graph_khop_jobs, self.h, seeds, ks, mode, threads)

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.lib.ref_graph_free(self.h)
            self.h = None

    def create_nodes(self, count):
        self.ref._check(self.ref.lib.ref_graph_create_nodes(self.h, count))

    def create_edge(self, src, relation, dst, props=""):
        if props:
            self.ref._check(self.ref.lib.ref_graph_create_edge_props(self.h, src, relation.encode(), dst,
                                                                     props.encode()))
        else:
            self.ref._check(self.ref.lib.ref_graph_create_edge(self.h, src, relation.encode(), dst))

    def create_node(self, labels="", props=""):
        self.ref._check(self.ref.lib.ref_graph_create_node_full(self.h, labels.encode(), props.encode()))

    def snapshot(self) -> bytes:
        """snapshot_to_string (snapshot.cpp:127-160): the reference's canonical text."""
        n = C.c_uint64()
        self.ref._check(self.ref.lib.ref_snapshot_to_string(self.h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        self.ref._check(self.ref.lib.ref_snapshot_to_string(self.h, buf, n.value + 1, C.byref(n)))
        return buf.raw[: n.value]

    @property
    def node_count(self):
        return int(self.ref.lib.ref_graph_node_count(self.h))

    def relation_csr(self, relation=None):
        rel = relation.encode() if relation is not None else None
        nr, nz = C.c_uint64(), C.c_uint64()
        self.ref._check(self.ref.lib.ref_graph_relation_csr(self.h, rel, C.byref(nr), C.byref(nz), None, None))
        rp = np.zeros(nr.value + 1, np.uint64)
        ci = np.zeros(max(nz.value, 1), np.uint64)
        self.ref._check(self.ref.lib.ref_graph_relation_csr(self.h, rel, C.byref(nr), C.byref(nz),
                                                            rp.ctypes.data, ci.ctypes.data))
        return rp, ci[: nz.value].copy()

    def k_hop_count(self, seed, k, mode=EXACT, relation=None):
        out = C.c_uint64()
        rel = relation.encode() if relation is not None else None
        self.ref._check(self.ref.lib.ref_k_hop_count(self.h, seed, k, mode, rel, C.byref(out)))
        return int(out.value)

    def k_hop_frontier(self, seed, k, mode=EXACT, relation=None):
        rel = relation.encode() if relation is not None else None
        n = C.c_uint64()
        cap = max(self.node_count, 1)
        ids = np.zeros(cap, np.uint64)
        self.ref._check(self.ref.lib.ref_k_hop_frontier(self.h, seed, k, mode, rel, ids.ctypes.data, cap,
                                                        C.byref(n)))
        return ids[: n.value].copy()

    def k_hop_count_many(self, seeds, k, mode=EXACT, threads=1):
        seeds = np.ascontiguousarray(seeds, np.uint64)
        counts = np.zeros(len(seeds), np.uint64)
        el = C.c_double()
        self.ref._check(self.ref.lib.ref_k_hop_count_many(self.h, seeds.ctypes.data, len(seeds), k, mode,
                                                          threads, counts.ctypes.data, C.byref(el)))
        return counts, el.value

    def pick_seeds(self, n, rng_seed):
        out = np.zeros(max(n, 1), np.uint64)
        self.ref._check(self.ref.lib.ref_pick_seeds(self.h, n, rng_seed, out.ctypes.data))
        return out[:n].copy()

    def cypher(self, text):
        """The reference's own executor: the result table's wire text."""
        n = C.c_uint64()
        self.ref._check(self.ref.lib.ref_cypher(self.h, text.encode(), None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        self.ref._check(self.ref.lib.ref_cypher(self.h, text.encode(), buf, n.value + 1, C.byref(n)))
        return buf.value.decode()


class RefBfs:
    def __init__(self, ref: Ref, h):
        self.ref, self.h = ref, h

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.lib.ref_bfs_oracle_free(self.h)
            self.h = None

    def count(self, seed, k, mode=EXACT):
        out = C.c_uint64()
        self.ref._check(self.ref.lib.ref_bfs_oracle_count(self.h, seed, k, mode, C.byref(out)))
        return int(out.value)

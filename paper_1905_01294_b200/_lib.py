"""ctypes binding of the C ABI in include/mgk.h (libmgk.so, built in-tree).

There is no fallback: if the library is missing or no GPU is present, the
calls fail loudly (MgkError / OSError). The CPU oracle lives under oracle/
and is never imported from this package.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

PKG = Path(__file__).resolve().parent
# MGK_LIB_PATH: an alternative build of the same library (A/B runs of compile-time variants)
LIB_PATH = Path(os.environ.get("MGK_LIB_PATH") or PKG / "lib" / "libmgk.so")

MGK_OK, MGK_ECONTRACT, MGK_EHARNESS, MGK_ECUDA, MGK_ENOMEM, MGK_ERANGE, MGK_ESNAPSHOT = range(7)
ENGINE_AUTO, ENGINE_SINGLE, ENGINE_LANES = 0, 1, 2
MAX_HOPS = 32


class MgkLevel(C.Structure):
    _fields_ = [("frontier", C.c_uint64), ("vertices", C.c_uint64), ("edges", C.c_uint64),
                ("union_edges", C.c_uint64), ("scanned", C.c_uint64), ("candidates", C.c_uint64),
                ("runs", C.c_uint32), ("pull_runs", C.c_uint32), ("ns", C.c_uint64)]


class MgkStats(C.Structure):
    _fields_ = [("engine", C.c_uint32), ("lanes", C.c_uint32), ("batches", C.c_uint32),
                ("hops", C.c_uint32), ("grid", C.c_uint32), ("block", C.c_uint32),
                ("launches", C.c_uint32), ("path", C.c_uint32),
                ("kernel_ms", C.c_double), ("setup_ns", C.c_uint64), ("cleanup_ns", C.c_uint64),
                ("level", MgkLevel * (MAX_HOPS + 1))]

    def to_dict(self) -> dict:
        levels = []
        for h in range(0, self.hops + 1):
            L = self.level[h]
            levels.append({k: getattr(L, k) for k, _ in MgkLevel._fields_})
        return {"engine": {1: "single", 2: "lanes"}.get(self.engine, str(self.engine)),
                "lanes": self.lanes, "batches": self.batches, "hops": self.hops,
                "grid": self.grid, "block": self.block, "launches": self.launches,
                "path": {0: "l2_bitmaps", 1: "smem_k2"}.get(self.path, str(self.path)),
                "kernel_ms": self.kernel_ms,
                "setup_us": self.setup_ns / 1e3, "cleanup_us": self.cleanup_ns / 1e3,
                "levels": levels}


class MgkTuning(C.Structure):
    _fields_ = [("alpha", C.c_uint32), ("beta", C.c_uint32), ("force_dir", C.c_uint32),
                ("lanes_words", C.c_uint32), ("alpha_lanes", C.c_uint32), ("alpha_last", C.c_uint32)]


# (name, restype, argtypes) for every symbol include/mgk.h declares
_vp, _u64, _u32, _int = C.c_void_p, C.c_uint64, C.c_uint32, C.c_int
_u64p, _u32p = C.POINTER(C.c_uint64), C.POINTER(C.c_uint32)
SIGNATURES = [
    ("mgk_graph_upload", _int, [_int, _u64, _u64, _vp, _vp, C.POINTER(_vp)]),
    ("mgk_graph_upload_u32", _int, [_int, _u64, _u64, _vp, _vp, C.POINTER(_vp)]),
    ("mgk_graph_from_edges", _int, [_int, _u64, _u64, _vp, _vp, C.POINTER(_vp)]),
    ("mgk_graph_gen_rmat", _int, [_int, _u32, _u32, C.c_double, C.c_double, C.c_double, _u64, _u64, _int,
                                  C.POINTER(_vp)]),
    ("mgk_graph_load_snapshot", _int, [_int, C.c_char_p, _u64, C.c_char_p, C.POINTER(_vp), _u64p]),
    ("mgk_graph_load_snapshot_file", _int, [_int, C.c_char_p, C.c_char_p, C.POINTER(_vp), _u64p]),
    ("mgk_snapshot_check", _int, [C.c_char_p, _u64, _u64p, _u64p]),
    ("mgk_graph_free", _int, [_vp]),
    ("mgk_mxm", _int, [_int, _u64, _u64, _vp, _vp, _vp, _u64, _u64, _vp, _vp, _vp, _int, _u64, _u64, _vp, _vp,
                       C.POINTER(_vp)]),
    ("mgk_matrix_info", _int, [_vp, _u64p, _u64p, _u64p, C.POINTER(_int)]),
    ("mgk_matrix_download", _int, [_vp, _vp, _vp, _vp]),
    ("mgk_matrix_free", _int, [_vp]),
    ("mgk_graph_info", _int, [_vp, _u64p, _u64p, C.POINTER(_int)]),
    ("mgk_graph_download_csr", _int, [_vp, _vp, _vp]),
    ("mgk_graph_download_csc", _int, [_vp, _vp, _vp]),
    ("mgk_graph_device_bytes", _u64, [_vp]),
    ("mgk_khop_count", _int, [_vp, _vp, _u64, _u32, _int, _vp]),
    ("mgk_khop_count_ex", _int, [_vp, _vp, _u64, _u32, _int, _int, _vp, C.POINTER(MgkStats)]),
    ("mgk_khop_count_device", _int, [_vp, _vp, _u64, _u32, _int, _int, _vp, _vp]),
    ("mgk_khop_count_device_ks", _int, [_vp, _vp, _u64, _vp, _u32, _int, _vp, _vp]),
    ("mgk_khop_device_stats", _int, [_vp, _vp, C.POINTER(MgkStats)]),
    ("mgk_khop_device_check", _int, [_vp, _vp]),
    ("mgk_graph_replicate", _int, [_vp, _int, C.POINTER(_vp)]),
    ("mgk_graph_transpose", _int, [_vp, C.POINTER(_vp)]),
    ("mgk_khop_count_ks", _int, [_vp, _vp, _u64, _vp, _u32, _int, _vp]),
    ("mgk_khop_count_schedule", _int, [_vp, _vp, _vp, _vp, _u32, _int, _vp]),
    ("mgk_khop_count_device_schedule", _int, [_vp, _vp, _vp, _vp, _u32, _int, _vp, _vp]),
    ("mgk_khop_count_multi", _int, [_vp, _int, _vp, _u64, _u32, _int, _vp]),
    ("mgk_khop_frontier", _int, [_vp, _u64, _u32, _int, _vp, _u64, _u64p]),
    ("mgk_walk_count", _int, [_vp, _vp, _u64, _u32, _u32, _int, _vp]),
    ("mgk_walk_targets", _int, [_vp, _u64, _u32, _u32, _vp, _u64, _u64p]),
    ("mgk_graph_set_tuning", _int, [_vp, C.POINTER(MgkTuning)]),
    ("mgk_graph_get_tuning", _int, [_vp, C.POINTER(MgkTuning)]),
    ("mgk_last_error", C.c_char_p, []),
    ("mgk_abi_version", _int, []),
    ("mgk_device_count", _int, []),
    ("mgk_gen_rmat_csr", _int, [_u32, _u32, C.c_double, C.c_double, C.c_double, _u64, _u64, _int,
                                _int, _u64p, _u64p, _vp, _vp]),
    ("mgk_pick_seeds_csr", _int, [_u64, _vp, _u64, _u64, _vp]),
    ("mgk_snapshot_write_csr", _int, [_u64, _vp, _vp, C.c_char_p, _int, _vp, _u64, _u64p]),
]

_lib = None


def lib() -> C.CDLL:
    """Load libmgk.so (once). Raises OSError when it has not been built."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise OSError(f"{LIB_PATH} is missing: run `make` (or __graft_entry__.build()) first")
        L = C.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | getattr(os, "RTLD_GLOBAL", 0))
        for name, res, args in SIGNATURES:
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def last_error() -> str:
    return lib().mgk_last_error().decode()

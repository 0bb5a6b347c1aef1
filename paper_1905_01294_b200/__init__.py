"""B200-native k-hop neighbourhood count (drop-in for matgraph's k_hop_count path).

The compute lives in libmgk.so (hand-written sm_100a CUDA behind the C ABI in
include/mgk.h); this package is the Python host mirror of the reference's
interface (proj/core/include/matgraph/execute.hpp, bench.hpp). See DESIGN.md.
"""
from .khop import (  # noqa: F401
    ENGINE_AUTO, ENGINE_LANES, ENGINE_SINGLE, K_MAX_HOPS, ContractError, DeviceError, DeviceGraph, SnapshotError,
    snapshot_check, mxm, SEMIRING_BOOL_OR_AND, SEMIRING_PLUS_TIMES, SEMIRING_MIN_PLUS,
    Error, HarnessError, KHopQuery, TraverseMode, Tuning, device_check, device_count, device_stats, k_hop_count,
    k_hop_count_batch, k_hop_count_device, k_hop_count_device_schedule, k_hop_count_device_sections, k_hop_count_multi,
    k_hop_count_schedule, k_hop_count_sections, k_hop_frontier, walk_count_batch, walk_targets)

__version__ = "0.1.0"

import sys, time, ctypes as C
sys.path.insert(0, '.')
import numpy as np
from paper_1905_01294_b200 import DeviceGraph, harness as H, k_hop_count_sections, _lib
rp, ci = H.gen_csr(H.G2)
g = DeviceGraph.from_csr(rp, ci)
seeds = np.ascontiguousarray(H.pick_seeds(rp, 300, 1), np.uint64)
ks = np.array([1, 2], np.uint32)
out = np.empty((2, 300), np.uint64)
lib = _lib.lib()
for _ in range(20): k_hop_count_sections(g, seeds, [1, 2], 0)
def t(f, n=200):
    ts = []
    for _ in range(n):
        t0 = time.perf_counter(); f(); ts.append(time.perf_counter() - t0)
    return np.median(ts) * 1e6, np.min(ts) * 1e6
print("sections wrapper us (median, min)", t(lambda: k_hop_count_sections(g, seeds, [1, 2], 0)))
print("raw ctypes us", t(lambda: lib.mgk_khop_count_ks(g.handle, seeds.ctypes.data, 300, ks.ctypes.data, 2, 0, out.ctypes.data)))
print("k=1 only raw", t(lambda: lib.mgk_khop_count_ks(g.handle, seeds.ctypes.data, 300, ks.ctypes.data, 1, 0, out.ctypes.data)))

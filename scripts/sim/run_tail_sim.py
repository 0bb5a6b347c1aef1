"""Design probe: hub / tail share of the scanned entries (scripts/sim/tail_sim.c)."""
import ctypes as C, subprocess, sys, time
import numpy as np
sys.path.insert(0, '.')
import oracle
from paper_1905_01294_b200 import harness as H
spec = H.SPECS[sys.argv[1]]
P = oracle.Port()
t = time.time(); rp, ci = P.gen_spec(spec); print("gen", time.time() - t, flush=True)
n = len(rp) - 1
p = lambda a: a.ctypes.data_as(C.c_void_p)
cp = np.zeros(n + 1, np.uint32); ri = np.zeros(len(ci), np.uint32)
C.CDLL('scripts/sim/lane_sim.so').build_csc(C.c_uint64(n), p(rp), p(ci), p(cp), p(ri))
deg = np.diff(rp.astype(np.int64))
order = np.lexsort((np.arange(n), -deg))
rank = np.empty(n, np.uint32); rank[order] = np.arange(n, dtype=np.uint32)
seeds = P.pick_seeds_u32(rp, 10, 1).astype(np.uint32)
k = 6
for Hh in [int(x) for x in sys.argv[2:]] or [131072]:
    out = np.zeros((k, 6), np.uint64)
    C.CDLL('scripts/sim/tail_sim.so').tail_sim(C.c_uint64(n), p(rp), p(ci), p(cp), p(ri), p(seeds), 10, k, p(rank), C.c_uint32(Hh), p(out))
    print("H", Hh)
    for h in range(k):
        o = out[h]; sc = o[:4].sum()
        if sc: print(f"hop {h+1}: scanned {sc/1e6:8.2f}M hub_in {o[0]/1e6:.2f} hub_out {o[1]/1e6:.2f} tail_in {o[2]/1e6:.2f} tail_out {o[3]/1e6:.2f} |F| {o[4]/1e6:.2f}M full-scan verts {o[5]/1e6:.2f}M", flush=True)

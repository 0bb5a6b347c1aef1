"""Design probe: LANES pull cost per hop, all-lanes vs per-lane direction (scripts/sim/lane_sim.c)."""
import ctypes as C, sys, time
import numpy as np
sys.path.insert(0, '.')
import oracle
from paper_1905_01294_b200 import harness as H

class HC(C.Structure):
    _fields_ = [(f, C.c_uint64) for f in ("pull_all", "pull_lane", "push_lane", "push_all", "cand_all", "cand_lane")]

def csc_sorted(rp, ci):
    n = len(rp) - 1
    deg = np.diff(rp.astype(np.int64))
    src = np.repeat(np.arange(n, dtype=np.uint32), deg)
    # per column: descending out-degree of the source, ties ascending id
    order = np.lexsort((src, -deg[src], ci))
    ri = src[order].astype(np.uint32)
    cp = np.zeros(n + 1, np.uint32)
    np.cumsum(np.bincount(ci, minlength=n), out=cp[1:])
    return cp, ri

spec = H.SPECS[sys.argv[1]] if len(sys.argv) > 1 else H.G2
nseeds = int(sys.argv[2]) if len(sys.argv) > 2 else 10
alpha = int(sys.argv[3]) if len(sys.argv) > 3 else 4
P = oracle.Port()
t = time.time(); rp, ci = P.gen_spec(spec); print("gen", time.time() - t, flush=True)
cp = np.zeros(len(rp), np.uint32); ri = np.zeros(len(ci), np.uint32)
L0 = C.CDLL('scripts/sim/lane_sim.so'); L0.build_csc(C.c_uint64(len(rp) - 1), rp.ctypes.data_as(C.c_void_p), ci.ctypes.data_as(C.c_void_p), cp.ctypes.data_as(C.c_void_p), ri.ctypes.data_as(C.c_void_p)); print("csc", time.time() - t, flush=True)
seeds = P.pick_seeds_u32(rp, max(nseeds, 10), 1)[:nseeds].astype(np.uint32)
L = C.CDLL('scripts/sim/lane_sim.so')
out = (HC * 6)()
p = lambda a: a.ctypes.data_as(C.c_void_p)
L.lane_sim(C.c_uint64(len(rp) - 1), p(rp), p(ci), p(cp), p(ri), p(seeds), nseeds, 6, alpha, out)
for h in range(6):
    o = out[h]
    print(f"hop {h+1}: push_all {o.push_all/1e6:9.2f}M  pull_all {o.pull_all/1e6:9.2f}M (cand {o.cand_all/1e6:.2f}M)"
          f"  | perlane: push {o.push_lane/1e6:9.2f}M pull {o.pull_lane/1e6:9.2f}M (cand {o.cand_lane/1e6:.2f}M)")

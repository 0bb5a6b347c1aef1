"""Design probe: split-pull cost model (scripts/sim/hyb_sim.c) on G2 / G4. Build: gcc -O2 -shared -fPIC -o scripts/sim/hyb_sim.so scripts/sim/hyb_sim.c (and sortin.c, lane_sim.c)."""
import ctypes as C, sys, time
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
# in-lists by descending source out-degree (ties by id), like the device CSC
C.CDLL('scripts/sim/sortin.so').sort_in(C.c_uint64(n), p(cp), p(ri), p(rp))
seeds = P.pick_seeds_u32(rp, 10, 1).astype(np.uint32)
D = np.array([int(x) for x in sys.argv[2:]], np.uint32)
srt = np.sort(deg)[::-1]
for d in D: print("D", d, "hubs", int((deg >= d).sum()), "hub edge share", float(deg[deg >= d].sum() / deg.sum()))
k = 5
out = np.zeros((k, len(D), 3), np.uint64)
C.CDLL('scripts/sim/hyb_sim.so').hyb_sim(C.c_uint64(n), p(rp), p(ci), p(cp), p(ri), p(seeds), 10, k, p(D), len(D), p(out))
for h in range(k):
    print(f"hop {h+1}: all-pull {out[h,0,2]/1e6:.1f}M | " + " | ".join(f"D={D[i]}: pull {out[h,i,0]/1e6:.1f}M push {out[h,i,1]/1e6:.1f}M" for i in range(len(D))), flush=True)

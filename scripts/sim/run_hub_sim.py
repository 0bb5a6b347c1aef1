"""Design probe: hub-source share of the LANES pull's scanned entries (scripts/sim/hub_sim.c)."""
import ctypes as C, subprocess, sys, time
import numpy as np
sys.path.insert(0, '.')
import oracle
from paper_1905_01294_b200 import harness as H
subprocess.run("gcc -O2 -shared -fPIC -pthread -o scripts/sim/lane_sim.so scripts/sim/lane_sim.c && "
               "gcc -O2 -shared -fPIC -o scripts/sim/hub_sim.so scripts/sim/hub_sim.c", shell=True, check=True)
spec = H.SPECS[sys.argv[1]] if len(sys.argv) > 1 else H.G2
P = oracle.Port()
t = time.time(); rp, ci = P.gen_spec(spec); print("gen", time.time() - t, flush=True)
n = len(rp) - 1
p = lambda a: a.ctypes.data_as(C.c_void_p)
cp = np.zeros(n + 1, np.uint32); ri = np.zeros(len(ci), np.uint32)
C.CDLL('scripts/sim/lane_sim.so').build_csc(C.c_uint64(n), p(rp), p(ci), p(cp), p(ri))
deg = np.diff(rp.astype(np.int64))
order = np.lexsort((np.arange(n), -deg))
rank = np.empty(n, np.uint32); rank[order] = np.arange(n, dtype=np.uint32)
Hs = np.array([8192, 16384, 32768, 65536, 131072, 262144], np.uint32)
seeds = P.pick_seeds_u32(rp, 10, 1).astype(np.uint32)
k = 6
sc = np.zeros(k, np.uint64); fh = np.zeros(k, np.uint64); hh = np.zeros((k, len(Hs)), np.uint64)
C.CDLL('scripts/sim/hub_sim.so').hub_sim(C.c_uint64(n), p(rp), p(ci), p(cp), p(ri), p(seeds), 10, k, p(rank),
                                         p(Hs), len(Hs), p(sc), p(hh), p(fh))
for h in range(k):
    if sc[h]:
        print(f"hop {h+1}: scanned {sc[h]/1e6:9.2f}M  frontier-source share {fh[h]/sc[h]:.2f}  hub share " +
              " ".join(f"H={int(x)//1024}K:{hh[h,i]/sc[h]:.2f}" for i, x in enumerate(Hs)))

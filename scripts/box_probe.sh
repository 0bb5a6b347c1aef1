#!/bin/bash
# Host facts of the GPU box + a timing of the host-side G4 generator.
set -x
nproc; free -g; lscpu | head -20; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python - <<'PY'
import time, sys
sys.path.insert(0, '.')
from paper_1905_01294_b200 import harness as H
t = time.time(); rp, ci = H.gen_csr(H.G2); print("G2 host gen", time.time() - t, len(rp) - 1, len(ci), flush=True)
t = time.time(); rp, ci = H.gen_csr(H.G4); print("G4 host gen", time.time() - t, len(rp) - 1, len(ci), flush=True)
import resource; print("maxrss GB", resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 2**20)
PY

#!/bin/bash
mkdir -p gpurun_out
MGK_MS_DIAG=1 python scripts/lanes_probe.py both 16 > gpurun_out/ab_base.log 2>&1
MGK_F1_SEPARATE=1 MGK_MS_DIAG=1 python scripts/lanes_probe.py both 16 > gpurun_out/ab_sep.log 2>&1
MGK_L2_PERSIST=1 MGK_MS_DIAG=1 python scripts/lanes_probe.py both 16 > gpurun_out/ab_persist.log 2>&1
python -c "
import torch; p=torch.cuda.get_device_properties(0); print(p)
from cuda.bindings import runtime as rt
for a in ('cudaDevAttrMaxPersistingL2CacheSize','cudaDevAttrMaxAccessPolicyWindowSize','cudaDevAttrL2CacheSize'):
    print(a, rt.cudaDeviceGetAttribute(getattr(rt.cudaDeviceAttr, a), 0))
" > gpurun_out/ab_props.log 2>&1
bash scripts/r02_quick.sh
grep -h "k=6" gpurun_out/ab_*.log

#!/bin/bash
# A/B: out-degree ids with / without the predicated hub-word gathers
mkdir -p gpurun_out
export MGK_MS_DIAG=1
MGK_RELABEL=2 MGK_PROBE_HUB=1 timeout 600 python scripts/lanes_probe.py both 16 > gpurun_out/ab2_r2_nohub.log 2>&1
MGK_RELABEL=2 timeout 600 python scripts/lanes_probe.py both 16 > gpurun_out/ab2_r2_hub.log 2>&1
MGK_RELABEL=2 MGK_PROBE_HUB=8192 timeout 600 python scripts/lanes_probe.py both 16 > gpurun_out/ab2_r2_hub8k.log 2>&1
timeout 600 python scripts/lanes_probe.py both 16 > gpurun_out/ab2_base.log 2>&1
for f in gpurun_out/ab2_*.log; do echo "== $f"; grep -h "k=6\|Error" $f | cut -c1-400; done

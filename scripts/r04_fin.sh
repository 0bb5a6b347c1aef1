#!/bin/bash
# finalize: visited-lane masking inside the discovered-vertex block (the dense sweep's load block as before)
export MGK_MS_DIAG=1
timeout 600 python scripts/lanes_probe.py both 10 2>&1 | grep "k=6\|rror" | cut -c1-900
unset MGK_MS_DIAG
timeout 1500 python -m pytest -q -m gpu tests/test_gpu_configs.py tests/test_gpu_parity.py -x 2>&1 | tail -3

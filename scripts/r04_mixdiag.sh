#!/bin/bash
# mixed hop split: MGK_MS_DIAG puts the pull part's ns of a mixed hop in the last field (us)
export MGK_MS_DIAG=1
for s in 32 64 128; do echo "== strag $s"; MGK_STRAG=$s timeout 600 python scripts/lanes_probe.py G4 10 2>&1 | grep "bits=\|rror" | cut -c1-900; done

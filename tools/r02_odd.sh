#!/bin/bash
# A/B of the odd-pitch paths (tools/ab_odd.py, pipelined clock, parity-checked):
# padded scalar tile vs the cp.async-staged kernel at several ring depths / residencies.
for r in 1 2; do
  for t in "transpose.staged=0" "transpose.staged=1" "transpose.staged_stages=3" "transpose.staged_ctas=3" \
           "transpose.staged_ctas=1" "transpose.staged_stages=2,transpose.staged_ctas=3"; do
    B2K_TUNE="$t" timeout 300 python tools/ab_odd.py
  done
done

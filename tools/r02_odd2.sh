#!/bin/bash
# odd pitches: scalar tile vs the staged kernel forced, ring depth / residency / L2 evict-first hint
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for r in 1 2; do
  for t in "transpose.staged=0" "transpose.staged=2" "transpose.staged=2,transpose.staged_hint=1" \
           "transpose.staged=2,transpose.staged_stages=2,transpose.staged_ctas=3" \
           "transpose.staged=2,transpose.staged_stages=2,transpose.staged_ctas=3,transpose.staged_hint=1" \
           "transpose.staged=2,transpose.staged_stages=2,transpose.staged_ctas=4" \
           "transpose.staged=2,transpose.staged_stages=3,transpose.staged_hint=1"; do
    B2K_TUNE="$t" timeout 300 python tools/ab_odd.py
  done
done

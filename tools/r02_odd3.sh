#!/bin/bash
# odd pitches: scalar tile vs staged kernel geometries (64 / 128 / 256-row tiles, hint)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for r in 1 2; do
  for t in "transpose.staged=0" "transpose.staged=1" "transpose.staged=2,transpose.staged_geom=6" "transpose.staged=2,transpose.staged_geom=1" \
           "transpose.staged=2,transpose.staged_geom=2" "transpose.staged=2,transpose.staged_geom=3" \
           "transpose.staged=2,transpose.staged_geom=4" "transpose.staged=2,transpose.staged_geom=5"; do
    B2K_TUNE="$t" timeout 300 python tools/ab_odd.py
  done
done

#!/bin/bash
# odd pitches: more staged geometries around the 128-row tiles (3 CTAs, 192 rows, 3 stages)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for r in 1 2; do
  for t in "transpose.staged=1" "transpose.staged=2,transpose.staged_geom=7" "transpose.staged=2,transpose.staged_geom=8" "transpose.staged=2,transpose.staged_geom=9"; do
    B2K_TUNE="$t" timeout 300 python tools/ab_odd.py
  done
done

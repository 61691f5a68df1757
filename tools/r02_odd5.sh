#!/bin/bash
# odd pitches: 512-B staged row runs (geometries 7 / 8) vs the auto geometry
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for r in 1 2; do
  for t in "transpose.staged=1" "transpose.staged=2,transpose.staged_geom=7" "transpose.staged=2,transpose.staged_geom=8"; do
    B2K_TUNE="$t" timeout 300 python tools/ab_odd.py
  done
done

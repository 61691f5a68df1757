#!/bin/bash
# bench step A/B: LDG transpose vs cp.async (no hint / L2 evict-first policy / 256-B prefetch), interleaved
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for r in 1 2 3; do
  for t in "transpose.cpa=0" "transpose.cpa=1" "transpose.cpa_hint=1" "transpose.cpa_hint=2"; do
    B2K_TUNE=$t timeout 600 python bench.py --no-e2e --no-cpu > gpurun_out/j21_bench_$t.$r.json 2> gpurun_out/j21.err
  done
done

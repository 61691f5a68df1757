#!/bin/bash
# bench step A/B: reduction loads with / without the L2 evict-first policy; C2 probe
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for r in 1 2 3; do
  for t in "reduce.hint=0" "reduce.hint=1"; do
    B2K_TUNE=$t timeout 600 python bench.py --no-e2e --no-cpu > gpurun_out/j34_bench_$t.$r.json 2>> gpurun_out/j34.err
  done
done
for t in 0 1; do echo "hint=$t $(B2K_TUNE=reduce.hint=$t timeout 300 python tools/r02_c2_probe.py)"; done > gpurun_out/j34_c2.log

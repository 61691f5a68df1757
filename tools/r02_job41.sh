#!/bin/bash
# bench step A/B with the cp.async transpose: reduction variants (128-bit default vs 256-bit loads)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for r in 1 2 3; do
  for t in "reduce.variant=0" "reduce.variant=5" "reduce.variant=6" "reduce.variant=9"; do
    B2K_TUNE=$t timeout 600 python bench.py --no-e2e --no-cpu > gpurun_out/j41_bench_$t.$r.json 2>> gpurun_out/j41.err
  done
done

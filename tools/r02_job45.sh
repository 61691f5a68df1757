#!/bin/bash
# C2 (2^24) reduce_sum residency / loads-in-flight sweep (CUDA graph over rotating inputs)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for t in "reduce.ctas_per_sm=2" "reduce.ctas_per_sm=3" "reduce.ctas_per_sm=4" "reduce.variant=1" "reduce.variant=1,reduce.ctas_per_sm=4" "reduce.variant=3,reduce.ctas_per_sm=2" "reduce.variant=2,reduce.ctas_per_sm=8" "reduce.variant=4,reduce.ctas_per_sm=8"; do
  echo "$t $(B2K_TUNE=$t timeout 300 python tools/r02_c2_probe.py)"
done

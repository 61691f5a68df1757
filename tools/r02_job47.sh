#!/bin/bash
# C2 tail probe: reduce_sum as shipped vs builds without the grid combine (block partials)
# and without the block tree (warp trees only); results of the probes are not sums
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for r in 1 2; do
  for lib in paper_2605_13864_b200/libb200k.so abtest/libprobe2.so abtest/libprobe1.so; do
    echo "$lib $(B2K_LIB=$PWD/$lib timeout 300 python tools/r02_c2_probe.py)"
  done
done

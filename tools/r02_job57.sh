#!/bin/bash
# cp.async transpose store cache hint A/B in the bench step (builds under abtest/)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for r in 1 2 3; do
  for lib in paper_2605_13864_b200/libb200k.so abtest/libstnormal.so abtest/libstlast.so; do
    echo "$lib $(B2K_LIB=$PWD/$lib timeout 600 python bench.py --no-e2e --no-cpu | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["value"]), round(d["kernels"]["transpose"]["GBps"]), round(d["kernels"]["reduce"]["GBps"]))')"
  done
done

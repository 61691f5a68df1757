#!/bin/bash
# ncu --set full of the cp.async transpose variants vs the LDG path at C4
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for v in 0 3 ldg; do
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:transpose_(cpa|vec)" -s 2 -c 1 \
     -o gpurun_out/j15_cpa_$v -f python tools/prof_cpa.py $v > gpurun_out/j15_ncu_$v.log 2>&1
done
ls -la gpurun_out

#!/bin/bash
# cp.async default with the evict-first hint: full check, ncu of the bench command,
# isolated geometry A/B, e2e A/B against the LDG path
bash tools/r02_check.sh
bash tools/ncu_bench.sh
timeout 900 python tools/r02_cpa.py ldg,auto,auto_nohint,cpa2,cpa5 > gpurun_out/j22_cpa.jsonl 2> gpurun_out/j22_cpa.err
for r in 1 2; do
  for c in 0 1; do
    B2K_TUNE=transpose.cpa=$c timeout 600 python bench.py --no-cpu > gpurun_out/j22_bench_e2e_cpa$c.$r.json 2> gpurun_out/j22_e2e.err
  done
done

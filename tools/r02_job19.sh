#!/bin/bash
# cp.async geometry A/B (incl. auto) + bench step with the LDG vs cp.async transpose, interleaved
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python tools/r02_cpa.py ldg,auto,cpa2,cpa5,cpa8,cpa9 > gpurun_out/j19_cpa.jsonl 2> gpurun_out/j19_cpa.err
for r in 1 2 3; do
  for c in 0 1; do
    B2K_TUNE=transpose.cpa=$c timeout 600 python bench.py --no-e2e --no-cpu > gpurun_out/j19_bench_cpa$c.$r.json 2> gpurun_out/j19_bench_cpa$c.$r.err
  done
done

#!/bin/bash
# two-level ticket grid combine: C2 probe across group counts + reduction tests with it on
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for r in 1 2; do
  for t in "reduce.groups=0" "reduce.groups=4" "reduce.groups=8" "reduce.groups=15"; do
    echo "$t $(B2K_TUNE=$t timeout 300 python tools/r02_c2_probe.py)"
  done
done > gpurun_out/j48_c2.log 2>&1
for r in 1 2; do
  for t in "reduce.groups=0" "reduce.groups=8" "reduce.groups=15"; do
    B2K_TUNE=$t timeout 600 python bench.py --no-e2e --no-cpu > gpurun_out/j48_bench_$t.$r.json 2>> gpurun_out/j48.err
  done
done
B2K_TUNE=reduce.groups=15 timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_fused_combine.py tests/test_gpu_multi.py tests/test_gpu_fullsize.py tests/test_gpu_threads.py tests/test_gpu_interp.py -x -q > gpurun_out/j48_pytest.log 2>&1; tail -2 gpurun_out/j48_pytest.log

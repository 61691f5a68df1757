#!/bin/bash
# A/B of two library builds (abtest/libold.so = HEAD before the 2-byte row-pair mapping)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for r in 1 2; do
  for lib in abtest/libold.so paper_2605_13864_b200/libb200k.so; do
    for t in "transpose.staged=1" "transpose.staged=2,transpose.staged_geom=6"; do
      B2K_LIB=$PWD/$lib B2K_TUNE="$t" timeout 300 python tools/ab_odd.py
    done
  done
done > gpurun_out/j42_odd.jsonl 2> gpurun_out/j42.err
timeout 300 ncu --metrics gpu__time_duration.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum --clock-control none --csv -k "regex:transpose_staged" -c 1 -s 2 python tools/prof_odd_default.py bf16 16385 16383 > gpurun_out/j42_ncu.csv 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "staged or unaligned or sweep" > gpurun_out/j42_pytest.log 2>&1; tail -2 gpurun_out/j42_pytest.log

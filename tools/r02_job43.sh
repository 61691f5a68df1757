#!/bin/bash
# 2-byte staged kernel: row-pair reads + 32-bit stores vs 32-row reads + 16-bit stores
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "row_pairs or staged_geometries" > gpurun_out/j43_pytest.log 2>&1; tail -2 gpurun_out/j43_pytest.log
for r in 1 2; do
  for t in "transpose.staged=1" "transpose.staged=1,transpose.staged_pair=1" "transpose.staged=2,transpose.staged_geom=6" "transpose.staged=2,transpose.staged_geom=6,transpose.staged_pair=1"; do
    B2K_TUNE="$t" timeout 300 python tools/ab_odd.py
  done
done > gpurun_out/j43_odd.jsonl 2> gpurun_out/j43.err
B2K_TUNE=transpose.staged_pair=1 timeout 300 ncu --metrics gpu__time_duration.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed.sum --clock-control none --csv -k "regex:transpose_staged" -c 1 -s 2 python tools/prof_odd_default.py bf16 16385 16383 > gpurun_out/j43_ncu.csv 2>&1

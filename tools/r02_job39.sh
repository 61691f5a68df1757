#!/bin/bash
# staged odd-pitch kernel with the per-width row rotation: A/B via ab_odd + ncu conflicts + tests
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for r in 1 2; do
  for t in "transpose.staged=0" "transpose.staged=1" "transpose.staged=2,transpose.staged_geom=6" "transpose.staged=2,transpose.staged_geom=1" "transpose.staged=2,transpose.staged_geom=4"; do
    B2K_TUNE="$t" timeout 300 python tools/ab_odd.py
  done
done > gpurun_out/j39_odd.jsonl 2> gpurun_out/j39.err
for d in f32 f64; do
  timeout 300 ncu --metrics gpu__time_duration.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum --clock-control none --csv -k "regex:transpose_staged" -c 1 -s 2 python tools/prof_odd_default.py $d 16385 16383 > gpurun_out/j39_ncu_$d.csv 2>&1
done
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "staged or unaligned" > gpurun_out/j39_pytest.log 2>&1; tail -2 gpurun_out/j39_pytest.log

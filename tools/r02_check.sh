#!/bin/bash
# Round-2 GPU check (one gpurun call): build, GPU tests (fp32 parity log), smoke,
# both bench arms, interleaved A/B of old/new library builds, shared-memory
# bank-conflict metrics of the bench transpose.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
rm -f gpurun_out/fp32_parity.jsonl
B2K_PARITY_LOG=$PWD/gpurun_out/fp32_parity.jsonl timeout 1800 python -m pytest tests/ -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?" >> gpurun_out/bench_ref.err
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --kernel-name-base demangled -k "regex:transpose_(vec|cpa)_kernel" -c 2 --log-file gpurun_out/ncu_conflicts.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-graph > gpurun_out/ncu_conflicts.log 2>&1

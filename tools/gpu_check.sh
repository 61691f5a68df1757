#!/bin/bash
# One gpurun call: build check, GPU tests, smoke, bench, ncu launch list + full capture.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/prof_run.py > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:transpose_vec -s 1 -c 1 -o gpurun_out/prof_transpose -f python tools/prof_run.py > gpurun_out/ncu_t.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:reduce_kernel -s 1 -c 1 -o gpurun_out/prof_reduce -f python tools/prof_run.py > gpurun_out/ncu_r.log 2>&1
ls -la gpurun_out

#!/bin/bash
# ncu evidence for the bench command itself: launch list (time + DRAM bytes) and
# one --set full capture per hot kernel, all from `python bench.py`.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:b2::.*transpose_(vec|cpa)_kernel" -s 2 -c 1 -o gpurun_out/prof_transpose -f $CMD > gpurun_out/ncu_t.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:b2::.*reduce_kernel<int" -s 2 -c 1 -o gpurun_out/prof_reduce -f $CMD > gpurun_out/ncu_r.log 2>&1
tail -n 2 gpurun_out/ncu_launch.log gpurun_out/ncu_t.log gpurun_out/ncu_r.log

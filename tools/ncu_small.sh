#!/bin/bash
# Cold-L2 (ncu --cache-control all) per-launch durations of the latency-bound cases.
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size \
    --clock-control none --kernel-name-base demangled -k "regex:b2::" --csv \
    --log-file gpurun_out/small_launches.csv python tools/small_kernels.py > gpurun_out/ncu_small.log 2>&1
echo "ncu rc=$?"

#!/bin/bash
# gpurun: knob sweep + bench (GPU-side numbers for tuning decisions)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python tools/tune.py > gpurun_out/tune.log 2>&1; echo "tune rc=$?" >> gpurun_out/tune.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log

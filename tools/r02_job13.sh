#!/bin/bash
# cp.async transpose A/B + generated-kernel coarsening / packing sweep + codegen GPU tests
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_codegen.py -x -q > gpurun_out/j13_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/j13_pytest.log
timeout 900 python tools/r02_cpa.py > gpurun_out/j13_cpa.jsonl 2> gpurun_out/j13_cpa.err
timeout 900 python tools/r02_codegen_kernels.py > gpurun_out/j13_codegen.jsonl 2> gpurun_out/j13_codegen.err
tail -3 gpurun_out/j13_pytest.log

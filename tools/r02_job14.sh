#!/bin/bash
# cp.async transpose (paired 256-bit stores) A/B + generated-kernel packing + codegen GPU tests
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_codegen.py tests/test_gpu_codegen_fuzz.py -x -q > gpurun_out/j14_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/j14_pytest.log
timeout 900 python tools/r02_cpa.py > gpurun_out/j14_cpa.jsonl 2> gpurun_out/j14_cpa.err
timeout 900 python tools/r02_codegen_kernels.py 4x1,8x2 > gpurun_out/j14_codegen.jsonl 2> gpurun_out/j14_codegen.err
tail -3 gpurun_out/j14_pytest.log

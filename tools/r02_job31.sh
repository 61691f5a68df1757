#!/bin/bash
# binary32 single ops in generated kernels: codegen GPU tests + fuzz + kernel bench
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_codegen.py tests/test_gpu_codegen_fuzz.py tests/test_gpu_families.py -x -q > gpurun_out/j31_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/j31_pytest.log
timeout 900 python tools/r02_codegen_kernels.py 4x1,8x2 > gpurun_out/j31_codegen.jsonl 2> gpurun_out/j31_codegen.err
tail -3 gpurun_out/j31_pytest.log

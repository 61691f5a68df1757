#!/bin/bash
# paired 64-bit loads in generated kernels: codegen GPU tests + kernel bench
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests/test_gpu_codegen.py tests/test_gpu_codegen_fuzz.py tests/test_gpu_codegen_scale.py tests/test_gpu_codegen_pipe.py tests/test_gpu_families.py -x -q > gpurun_out/j51_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/j51_pytest.log
timeout 900 python tools/r02_codegen_kernels.py 4x1,8x2 > gpurun_out/j51_codegen.jsonl 2> gpurun_out/j51_codegen.err
tail -3 gpurun_out/j51_pytest.log

#!/bin/bash
# pipeline lanes: thread / host-path tests (copy pool serialised)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_threads.py tests/test_gpu_kernels.py tests/test_gpu_interp.py tests/test_gpu_codegen.py -x -q > gpurun_out/j24_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/j24_pytest.log
tail -3 gpurun_out/j24_pytest.log

#!/bin/bash
# odd-pitch auto dispatch (staged 128-row tiles beyond 256 MB) vs scalar / old staged; tests
bash tools/r02_odd3.sh > gpurun_out/j36_odd.jsonl 2> gpurun_out/j36.err
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_fullsize.py -q -x > gpurun_out/j36_pytest.log 2>&1
tail -2 gpurun_out/j36_pytest.log

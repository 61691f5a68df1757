#!/bin/bash
# pipeline lanes: thread / host-path tests, e2e concurrent vs serial A/B
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_threads.py tests/test_gpu_kernels.py tests/test_gpu_interp.py -x -q > gpurun_out/j23_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/j23_pytest.log
for r in 1 2; do
  timeout 600 python bench.py --no-cpu > gpurun_out/j23_conc.$r.json 2> gpurun_out/j23.err
  timeout 600 python bench.py --no-cpu --e2e-serial > gpurun_out/j23_serial.$r.json 2>> gpurun_out/j23.err
done
tail -2 gpurun_out/j23_pytest.log

mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_props.py tests/test_gpu_sanitizer.py -q -x > gpurun_out/pytest_staged.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_staged.log
timeout 1500 bash tools/r02_odd.sh > gpurun_out/odd_ab.jsonl 2>&1
tail -3 gpurun_out/pytest_staged.log; cat gpurun_out/odd_ab.jsonl

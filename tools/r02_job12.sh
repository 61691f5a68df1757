mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_codegen.py tests/test_gpu_codegen_fuzz.py tests/test_gpu_codegen_pipe.py tests/test_gpu_codegen_scale.py tests/test_gpu_families.py -q -x > gpurun_out/pytest_tail.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_tail.log
timeout 900 python tools/r02_codegen_kernels.py > gpurun_out/codegen_kernels.jsonl 2> gpurun_out/codegen_kernels.err
tail -5 gpurun_out/pytest_tail.log; cat gpurun_out/codegen_kernels.jsonl; tail -3 gpurun_out/codegen_kernels.err

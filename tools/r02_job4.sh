mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_codegen_pipe.py tests/test_gpu_codegen.py tests/test_gpu_codegen_fuzz.py tests/test_gpu_codegen_scale.py tests/test_gpu_threads.py tests/test_gpu_kernels.py -q -x > gpurun_out/pytest_pipe.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_pipe.log
timeout 900 python tools/r02_codegen_e2e.py > gpurun_out/codegen_e2e.jsonl 2> gpurun_out/codegen_e2e.err
tail -30 gpurun_out/pytest_pipe.log; cat gpurun_out/codegen_e2e.jsonl; tail -5 gpurun_out/codegen_e2e.err

mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python tools/r02_pdl.py > gpurun_out/pdl.jsonl 2> gpurun_out/pdl.err
B2K_TUNE=launch.pdl=1 timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_multi.py tests/test_gpu_fused_combine.py -q -x > gpurun_out/pytest_pdl.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_pdl.log
timeout 900 python tools/r02_codegen_e2e.py > gpurun_out/codegen_e2e.jsonl 2> gpurun_out/codegen_e2e.err
cat gpurun_out/pdl.jsonl; tail -3 gpurun_out/pdl.err; tail -3 gpurun_out/pytest_pdl.log; cat gpurun_out/codegen_e2e.jsonl

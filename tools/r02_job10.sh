mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_codegen.py tests/test_gpu_codegen_fuzz.py tests/test_gpu_codegen_pipe.py tests/test_gpu_codegen_scale.py tests/test_gpu_families.py tests/test_gpu_interp.py tests/test_gpu_threads.py -q -x > gpurun_out/pytest_ix.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_ix.log
for ix in 0 1; do B2K_CODEGEN_IX32=$ix timeout 900 python tools/r02_codegen_kernels.py > gpurun_out/codegen_kernels_ix$ix.jsonl 2> gpurun_out/codegen_kernels_ix$ix.err; done
tail -15 gpurun_out/pytest_ix.log; cat gpurun_out/codegen_kernels_ix1.jsonl; tail -3 gpurun_out/codegen_kernels_ix1.err

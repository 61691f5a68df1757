mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python tools/r02_ragged.py > gpurun_out/ragged.jsonl 2>&1
B2K_PARITY_LOG=$PWD/gpurun_out/fp32_parity.jsonl timeout 2400 python -m pytest tests/ -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/ragged.jsonl

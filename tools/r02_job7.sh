mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python tools/r02_pdl.py > gpurun_out/pdl.jsonl 2> gpurun_out/pdl.err
cat gpurun_out/pdl.jsonl; tail -3 gpurun_out/pdl.err

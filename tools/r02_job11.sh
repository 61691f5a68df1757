mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python tools/r02_prof_a5.py > /dev/null 2>&1
python tools/r02_prof_a5.py transpose_gpu.optc > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:b2g_kernel -c 1 -o gpurun_out/prof_gen_a5 -f python tools/r02_prof_a5.py > gpurun_out/ncu_gen_a5.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:b2g_kernel -c 1 -o gpurun_out/prof_gen_a4 -f python tools/r02_prof_a5.py transpose_gpu.optc > gpurun_out/ncu_gen_a4.log 2>&1
tail -3 gpurun_out/ncu_gen_a5.log gpurun_out/ncu_gen_a4.log

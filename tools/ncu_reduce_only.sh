mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:b2::.*reduce_kernel<int" -s 2 -c 1 -o gpurun_out/prof_reduce -f $CMD > gpurun_out/ncu_r.log 2>&1
tail -n 3 gpurun_out/ncu_r.log

#!/bin/bash
# grid-combine ticket A/B at latency-bound sizes (C2 probe) + reduce GPU tests with the new ticket
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for r in 1 2 3; do
  for t in 0 1; do
    echo "ticket=$t $(B2K_TUNE=reduce.ticket=$t timeout 300 python tools/r02_c2_probe.py)"
  done
done
B2K_TUNE=reduce.ticket=1 timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_fused_combine.py tests/test_gpu_multi.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -2

mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python tools/r02_pipe_sweep.py > gpurun_out/pipe_sweep.jsonl 2> gpurun_out/pipe_sweep.err
_B=1 B2K_PIPE_TRACE=1 timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import numpy as np, torch, paper_2605_13864_b200 as b2
from paper_2605_13864_b200 import programs
N=8192; tp=b2.parse_program(programs.TRANSPOSE_GPU)
a=torch.empty((N,N),dtype=torch.float32,pin_memory=True).numpy(); o=torch.empty((N,N),dtype=torch.float32,pin_memory=True).numpy()
inp={'in': b2.Array([N,N],a.reshape(-1),'float'),'out': b2.Array([N,N],o.reshape(-1),'float'),'W':N,'H':N}
for i in range(2): b2.run_program(tp,'transpose',inp,backend='codegen')
" > gpurun_out/pipe_trace.log 2>&1
timeout 900 python -m pytest tests/test_gpu_codegen_pipe.py -q -x > gpurun_out/pytest_pipe.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_pipe.log
cat gpurun_out/pipe_sweep.jsonl; tail -3 gpurun_out/pipe_sweep.err; tail -20 gpurun_out/pipe_trace.log; tail -3 gpurun_out/pytest_pipe.log

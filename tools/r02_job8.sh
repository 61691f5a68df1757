mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
bash tools/ncu_bench.sh
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:transpose_staged_kernel" -c 1 -o gpurun_out/prof_staged -f python -c "
import sys; sys.path.insert(0,'.')
import torch, paper_2605_13864_b200 as b2
a=torch.randint(-30000,30000,(16385,16383),dtype=torch.int16,device='cuda'); b2.transpose(a); torch.cuda.synchronize()" > gpurun_out/ncu_staged.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:transpose_scalar_kernel" -c 1 -o gpurun_out/prof_scalar16 -f python -c "
import sys; sys.path.insert(0,'.')
import torch, paper_2605_13864_b200 as b2
from paper_2605_13864_b200 import _lib
_lib.tune('transpose.staged', 0)
a=torch.randint(-30000,30000,(16385,16383),dtype=torch.int16,device='cuda'); b2.transpose(a); torch.cuda.synchronize()" > gpurun_out/ncu_scalar16.log 2>&1
ls -la gpurun_out/*.ncu-rep; tail -2 gpurun_out/ncu_staged.log

set -x; exec > >(tee gpurun_out/probe.log) 2>&1
nproc; lscpu | head -30; free -g; nvidia-smi; nvidia-smi topo -m; numactl -H 2>/dev/null | head; ulimit -l; cat /proc/meminfo | head -5
python -c "
import torch,time
x=torch.empty(1<<30,dtype=torch.uint8).pin_memory()
d=torch.empty(1<<30,dtype=torch.uint8,device='cuda')
for i in range(3):
  torch.cuda.synchronize();t=time.time();d.copy_(x,non_blocking=True);torch.cuda.synchronize();print('h2d GB/s',1/(time.time()-t))
  torch.cuda.synchronize();t=time.time();x.copy_(d,non_blocking=True);torch.cuda.synchronize();print('d2h GB/s',1/(time.time()-t))
t=time.time(); y=torch.empty(16<<30,dtype=torch.uint8).pin_memory(); print('pin 16GB s',time.time()-t)
"

# Box probe: host resources, PCIe link, pinned-copy bandwidth (one direction and both at once).
set -x; exec > >(tee gpurun_out/probe.log) 2>&1
nproc; lscpu | head -30; free -g; nvidia-smi; nvidia-smi topo -m; numactl -H 2>/dev/null | head; ulimit -l; cat /proc/meminfo | head -5
nvidia-smi -q | grep -A3 -i "link width\|PCIe Generation" | head -20
python - <<'PY'
import torch,time
n=1<<30
x=torch.empty(n,dtype=torch.uint8).pin_memory(); y=torch.empty(n,dtype=torch.uint8).pin_memory()
d=torch.empty(n,dtype=torch.uint8,device='cuda'); e=torch.empty(n,dtype=torch.uint8,device='cuda')
s1=torch.cuda.Stream(); s2=torch.cuda.Stream()
def tm(f):
  torch.cuda.synchronize();t=time.perf_counter();f();torch.cuda.synchronize();return time.perf_counter()-t
for i in range(3):
  print('h2d GB/s %.1f'%(n/tm(lambda: d.copy_(x,non_blocking=True))/1e9))
  print('d2h GB/s %.1f'%(n/tm(lambda: y.copy_(d,non_blocking=True))/1e9))
  def both():
    with torch.cuda.stream(s1): d.copy_(x,non_blocking=True)
    with torch.cuda.stream(s2): y.copy_(e,non_blocking=True)
  print('bidir total GB/s %.1f'%(2*n/tm(both)/1e9))
t=time.time(); z=torch.empty(32<<30,dtype=torch.uint8).pin_memory(); print('pin 32GB s',time.time()-t)
PY

"""Kernel microbenchmark: k_adam (and the plan) on an in-memory table where
every block is visible, so one step = Adam over all K blocks (no transfers
after the first batch).  Usage: python tools/kbench.py [n_blocks] [steps]"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import workload as W  # noqa: E402
from paper_2605_20150_b200 import tidegs as T  # noqa: E402

nb = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
mask_p = float(sys.argv[3]) if len(sys.argv) > 3 else -1.0
B = 4096
sc = W.Scene(nb * B, B)
big = np.zeros((1, 6, 4), np.float32)
big[0] = [[1, 0, 0, 1e6], [-1, 0, 0, 1e6], [0, 1, 0, 1e6], [0, -1, 0, 1e6], [0, 0, 1, 1e6],
          [0, 0, -1, 1e6]]
s = torch.cuda.Stream()
t0 = time.time()
tab = T.Table(T.make_config(sc.N, B, nb, moments=T.COLD_RESTART), sc.bounds(), fill=sc.fill_fn,
              stream=s.cuda_stream)
print(f"setup {time.time() - t0:.1f}s")
act = tab.activate(big)
W.synth_grads_cuda(act, B, sc.N, 42, 0, s.cuda_stream)
mask = None
if mask_p >= 0:
    mask = torch.zeros((tab.P, B // 32), dtype=torch.int32, device="cuda")
    W.synth_mask_cuda(mask.data_ptr(), act, B, sc.N, 43, 0, int(mask_p * 2**32), s.cuda_stream)
lr = np.full(59, 1e-3, np.float32)
tab.step_adam(lr, mask_ptr=mask.data_ptr() if mask is not None else None)
for _ in range(3):
    tab.activate(big)
    tab.step_adam(lr, mask_ptr=mask.data_ptr() if mask is not None else None)
torch.cuda.synchronize()
tab.set_profiling(True)
for _ in range(steps):
    tab.activate(big)
    tab.step_adam(lr, mask_ptr=mask.data_ptr() if mask is not None else None)
tm = tab.timing()
ms = tm["adam_ms"] / tm["adam_launches"]
rows = nb * B
print(f"k_adam: {ms:.3f} ms/launch, rows {rows}, {rows * 1652 / ms / 1e6:.1f} GB/s algorithmic; "
      f"prologue {tm['adam_prologue_ms'] / steps * 1e3:.1f} us; plan {tm['plan_ms'] / steps * 1e3:.1f} us")
tab.close()

# Development helper: time the cfg2 product in complex64 (python tools/c64.py)
import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1401_6238_b200 import batched, workloads
h, x = workloads.cfg2()
dh = torch.from_numpy(h.astype(np.complex64)).cuda(); dx = torch.from_numpy(x.astype(np.complex64)).cuda()
y = torch.empty((4096, 1024), dtype=torch.complex64, device="cuda")
f = lambda: batched.hankel_tvp_partial(dh, [dx, dx, dx], (1024,)*4, out=y)
for _ in range(3): f()
torch.cuda.synchronize()
s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(20): f()
e.record(); torch.cuda.synchronize()
ms = s.elapsed_time(e) / 20
print(f"cfg2 c64: {ms*1e3:.1f} us/step, {4096/ms/1e3:.2f} M products/s, {4096*49128/ms/1e6:.0f} GB/s")

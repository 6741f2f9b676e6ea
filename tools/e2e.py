# Development helper (run from the repo root: python tools/e2e.py): e2e host->host throughput vs chunk size.
import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1401_6238_b200 import batched, workloads
h, x = workloads.cfg2()
hp = torch.from_numpy(h).pin_memory(); xp = torch.from_numpy(x).pin_memory()
yp = torch.empty((4096, 1024), dtype=torch.complex128, pin_memory=True)
for chunk in (256, 512, 1024, 2048):
    for _ in range(2): batched.hankel_tvp_partial_host(hp, [xp, xp, xp], (1024,) * 4, out=yp, chunk=chunk)
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5): batched.hankel_tvp_partial_host(hp, [xp, xp, xp], (1024,) * 4, out=yp, chunk=chunk)
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 5
    print(f"chunk {chunk}: {ms:.2f} ms/step, {4096 / ms * 1e3 / 1e6:.3f} M products/s, H2D {335.3 / ms:.1f} GB/s")

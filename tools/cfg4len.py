# Development helper (run from the repo root: python tools/cfg4len.py ...); not part of the package or the tests.
import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1401_6238_b200 import batched, workloads
Hb, X = workloads.cfg4()
dH = torch.from_numpy(Hb).cuda()
dxv = torch.from_numpy(np.ascontiguousarray(np.transpose(X, (0, 2, 1)))).cuda().reshape(1024, -1)
ref = None
for fl in [None, (256, 192), (192, 256), (256, 256)]:
    f = lambda: batched.bhhb_tvp_partial(dH, [dxv, dxv], 3, (64,)*3, (64,)*3, fft_lens=fl)
    y = f(); torch.cuda.synchronize()
    if ref is None: ref = y
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(3): f()
    e.record(); torch.cuda.synchronize()
    print(fl, f"{s.elapsed_time(e)/3*1e3:.0f} us", "relerr", (torch.linalg.norm(y-ref)/torch.linalg.norm(ref)).item())

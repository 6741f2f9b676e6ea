# Development helper (python tools/hooi_loop.py): time the cfg5 HOOI loop and
# count factor updates that fell back to the SVD.  Not part of the package/tests.
import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1401_6238_b200 import batched, workloads, hooi
sig, U0, shape = workloads.cfg5(signals=256)
dsig = torch.from_numpy(sig).cuda(); dU0 = torch.from_numpy(U0).cuda()
spec = batched.hankel_spectrum(dsig, shape)
orig = torch.linalg.svd
calls = [0]
def svd_count(*a, **k):
    calls[0] += 1
    return orig(*a, **k)
torch.linalg.svd = svd_count
f = lambda: hooi.hooi_symmetric_batched(dsig, shape, 5, dU0, max_iter=50, spectrum=spec)
f(); torch.cuda.synchronize(); calls[0] = 0
s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
s.record(); f(); e.record(); torch.cuda.synchronize()
print(f"50 sweeps x 256 signals: {s.elapsed_time(e):.1f} ms, svd fallbacks {calls[0]}")

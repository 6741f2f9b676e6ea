# Development helper: where one HOOI sweep of the cfg5 loop spends its time
# (torch profiler, CUDA time per op), 256 signals.
import sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1401_6238_b200 import batched, hooi, workloads
sig, U0, shape = workloads.cfg5(signals=256)
dsig = torch.from_numpy(sig).cuda()
spec = batched.hankel_spectrum(dsig, shape)
U = torch.from_numpy(U0).cuda()[None].expand(256, -1, -1).contiguous()
for _ in range(3):
    U = hooi.hooi_symmetric_batched(dsig, shape, 5, U, max_iter=1, spectrum=spec)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    U = hooi.hooi_symmetric_batched(dsig, shape, 5, U, max_iter=5, spectrum=spec)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25))
s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
s.record()
U = hooi.hooi_symmetric_batched(dsig, shape, 5, U, max_iter=10, spectrum=spec)
e.record(); torch.cuda.synchronize()
print("per sweep ms", s.elapsed_time(e) / 10)
Mb = torch.randn(256, 2000, 25, dtype=torch.complex128, device="cuda")
for name, fn in [("leading_left_singular", lambda: hooi.leading_left_singular(Mb, 5)),
                 ("gram", lambda: Mb.mH @ Mb),
                 ("eigh", lambda: torch.linalg.eigh(Mb.mH @ Mb))]:
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s.record()
    for _ in range(10): fn()
    e.record(); torch.cuda.synchronize()
    print(name, "ms", s.elapsed_time(e) / 10)

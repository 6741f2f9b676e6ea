# Development helper (run from the repo root: python tools/hooi.py ...); not part of the package or the tests.
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_1401_6238_b200 import batched, workloads
from paper_1401_6238_b200.hooi import hooi_symmetric_batched, leading_left_singular
sig, U0, shape = workloads.cfg5(signals=256)
dsig = torch.from_numpy(sig).cuda(); dU0 = torch.from_numpy(U0).cuda()
spec = batched.hankel_spectrum(dsig, shape)
def t(fn, reps=3):
    fn(); torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize(); return s.elapsed_time(e) / reps
M = torch.randn(256, 2000, 25, dtype=torch.complex128, device='cuda')
print("svd batch 256x2000x25:", t(lambda: leading_left_singular(M, 5)), "ms")
print("qr  batch:", t(lambda: torch.linalg.qr(M)), "ms")
print("loop 5 sweeps:", t(lambda: hooi_symmetric_batched(dsig, shape, 5, dU0, max_iter=5, spectrum=spec), 1), "ms")
def gram_left(M, r):
    G = M.conj().transpose(-1, -2) @ M
    w, V = torch.linalg.eigh(G)
    V = V[..., -r:].flip(-1); s = torch.sqrt(w[..., -r:].flip(-1))
    return (M @ V) / s[..., None, :]
# accuracy on realistic T from the loop
from paper_1401_6238_b200.hooi import fix_phase_batched
Uc = dU0.conj()[None].expand(256, -1, -1).contiguous()
T = batched.times_matrices(spec, shape, [Uc, Uc], spectrum=True).reshape(256, 2000, 25)
Us = leading_left_singular(T, 5)
Ug = fix_phase_batched(gram_left(T, 5))
print("gram:", t(lambda: gram_left(T, 5)), "ms; max col err", (Us - Ug).abs().max().item(),
      "proj err", max(torch.linalg.norm(Us[i] @ Us[i].conj().T - Ug[i] @ Ug[i].conj().T).item() for i in range(256)))

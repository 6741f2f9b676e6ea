# Exercise every kernel variant once with small inputs, for compute-sanitizer
# (memcheck / racecheck / synccheck); results are also checked against the
# oracle so a run that "passes" the sanitizer but computes garbage is caught.
#   compute-sanitizer --tool racecheck python tools/sanitize.py
# Development helper, not part of the package or the tests.
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import hankel_oracle as O  # noqa: E402
from paper_1401_6238_b200 import batched  # noqa: E402

rng = np.random.default_rng(0)
worst = 0.0


def rv(*shape, real=False):
    a = rng.standard_normal(shape)
    return a if real else a + 1j * rng.standard_normal(shape)


def check(name, got, ref, tol=1e-10):
    global worst
    err = float(np.linalg.norm(got - ref) / np.linalg.norm(ref))
    worst = max(worst, err if tol == 1e-10 else 0.0)
    print(f"{name:44s} rel err {err:.2e}", flush=True)
    assert err <= tol, name


def partial(shape, B, real=False, c64=False):
    d = sum(shape) - len(shape) + 1
    h = rv(B, d, real=real)
    x = rv(B, shape[1], real=real)
    dt = (np.float32 if real else np.complex64) if c64 else None
    hh, xx = (h.astype(dt), x.astype(dt)) if c64 else (h, x)
    dh, dx = torch.from_numpy(hh).cuda(), torch.from_numpy(xx).cuda()
    y = batched.hankel_tvp_partial(dh, [dx] * (len(shape) - 1), shape).cpu().numpy()
    c = lambda a: a.astype(np.complex128)
    ref = O.hankel_tvp_partial_batch(c(hh), [c(xx)] * (len(shape) - 1), shape)
    return y, ref


# k_small (latency kernel): a few products, L <= 4096
check("k_small  cfg1 shape, B=2", *partial((100,) * 3, 2, real=True))
# k_hankel_pp (TMA + mbarrier ping-pong, TMEM): cfg2 shape
check("k_hankel_pp  (1024,)^4, B=300", *partial((1024,) * 4, 300))
# k_hankel_fast with cp.async staging + WarpSync groups (L = 256, T = 16)
check("k_hankel_fast STG/WarpSync  (80,)^3, B=200", *partial((80,) * 3, 200))
# k_hankel_fast, L = 6144 / 8192 / 1024
check("k_hankel_fast L=6144  (2000,)^3, B=40", *partial((2000,) * 3, 40))
check("k_hankel_fast L=8192  (2700,)^3, B=40", *partial((2700,) * 3, 40))
check("k_hankel_fast L=1024  (300,)^3, B=64", *partial((300,) * 3, 64))
# generic k_hankel_1d (L = 768)
check("k_hankel_1d L=768  (250,)^3, B=64", *partial((250,) * 3, 64))
# four-step: packed real column pass (ST_A_PAIR) + Hermitian half
check("k_cols PAIR/half  real (5000,)^3, B=1", *partial((5000,) * 3, 1, real=True))
check("k_cols complex four-step  (5000,)^3, B=2", *partial((5000,) * 3, 2))
# 2D block plan (BHHB two-level)
Hg = rv(2, 118, 148)
X = rv(2, 40, 50)
dH = torch.from_numpy(Hg).cuda()
dx = torch.from_numpy(np.ascontiguousarray(np.transpose(X, (0, 2, 1)))).cuda().reshape(2, -1)
yb = batched.bhhb_tvp_partial(dH, [dx, dx], 3, (40,) * 3, (50,) * 3).cpu().numpy()
check("k_cols 2D block  BHHB 40x50 blocks, B=2", yb,
      O.bhhb_tvp_partial_batch(Hg, X, (40,) * 3, (50,) * 3))
# times_matrices combos (fast kernel combo table, column spectra)
h = rv(3, 5998)
M = rv(3, 2000, 4)
T = batched.times_matrices(torch.from_numpy(h).cuda(), (2000,) * 3,
                           [torch.from_numpy(M).cuda()] * 2).cpu().numpy()
check("times_matrices combos  (2000,)^3 r=4, B=3", T[1],
      O.times_matrices_fast(h[1], (2000,) * 3, [M[1], M[1]]))
# full products (deterministic reductions)
d = 3 * 99 + 1
h1, x1 = rv(40, d), rv(40, 100)
a = batched.hankel_tvp_full(torch.from_numpy(h1).cuda(), [torch.from_numpy(x1).cuda()] * 3,
                            (100,) * 3).cpu().numpy()
check("tvp_full  (100,)^3, B=40", a,
      np.array([O.hankel_tvp_full(h1[b], (100,) * 3, [x1[b]] * 3) for b in range(40)]))
# complex64 fast kernel and generic c64 kernel
check("k_hankel_fast_c64 (1024,)^4, B=300", *partial((1024,) * 4, 300, c64=True), tol=1e-4)
check("k_hankel_c64 L=768 (250,)^3, B=64", *partial((250,) * 3, 64, c64=True), tol=1e-4)
torch.cuda.synchronize()
print(f"all kernel variants ran; worst complex128 rel err {worst:.2e}")

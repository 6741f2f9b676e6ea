# Development helper (run from the repo root: python tools/lencheck.py ...); not part of the package or the tests.
import sys, numpy as np, torch
sys.path.insert(0, '.')
from oracle import hankel_oracle as O
from paper_1401_6238_b200 import batched
rng = np.random.default_rng(7)
for d in [200, 256, 500, 512, 1000, 1024, 2000, 2048, 3000, 4093, 4096, 6000, 8000]:
    for m in (2, 3):
        n1 = max(1, d // m); shape = [n1] + [(d - 1 + m - n1) // (m - 1)] * (m - 1)
        shape[-1] += d - (sum(shape) - m + 1)
        B = 3
        h = rng.standard_normal((B, d)) + 1j * rng.standard_normal((B, d))
        xs = [rng.standard_normal((B, n)) + 1j * rng.standard_normal((B, n)) for n in shape[1:]]
        y = batched.hankel_tvp_partial(torch.from_numpy(h).cuda(), [torch.from_numpy(x).cuda() for x in xs], shape).cpu().numpy()
        ref = np.stack([O.hankel_tvp_partial(h[b], shape, [x[b] for x in xs]) for b in range(B)])
        err = np.linalg.norm(y - ref) / np.linalg.norm(ref)
        print(f"d={d} m={m} shape={shape} err={err:.2e}", "FAIL" if err > 1e-12 else "")

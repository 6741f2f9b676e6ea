# Development helper: packed-real four-step products at the 256-row block edges, TMA vs generic column kernel.
import os, sys
sys.path.insert(0, ".")
import numpy as np, torch
from oracle import hankel_oracle as O
from paper_1401_6238_b200 import batched
for shape in [(7_500_000, 500_000, 500_000), (5_000_000, 1 << 21, 1 << 21), (4_500_000, 2_000_000, 2_000_000)]:
    rng = np.random.default_rng(shape[1] % 1000)
    d = sum(shape) - 2
    h = rng.standard_normal(d); x = rng.uniform(-1.0, 1.0, shape[1])
    ref = O.hankel_tvp_partial_padded(h, shape, [x, x], length=1 << 24)
    for env in ["", "HK_NO_COLTMA", "HK_NO_HALF", "HK_NO_PAIR"]:
        if env: os.environ[env] = "1"
        y = batched.hankel_tvp_partial(torch.from_numpy(h).cuda()[None], [torch.from_numpy(x).cuda()[None]] * 2, shape)[0].cpu().numpy()
        if env: os.environ.pop(env)
        err = np.abs(y - ref)
        bad = np.nonzero(err > 1e-8 * np.abs(ref).max())[0]
        print(shape, env or "default", "relerr", np.linalg.norm(y - ref) / np.linalg.norm(ref), "bad", len(bad), bad[:6], bad[-3:] if len(bad) else "")

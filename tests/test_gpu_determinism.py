"""Race / indexing checks in place of compute-sanitizer (closed on this GPU pool):

* every product is independent, so item b's output must be BITWISE identical
  whatever batch it is launched in (its position in the persistent grid, the
  tail of the last wave, the ping-pong slot of the TMA kernel, the staging
  slot of the cp.async kernel all change with the batch offset and size) --
  a shared-memory race, a missing barrier or a stale TMEM/staging slot shows
  up as a bit difference;
* repeated launches are bitwise identical (schedule independence, SPEC.md);
* outputs are written into NaN-poisoned buffers: every element must be
  overwritten and nothing outside the output rows touched.
Covers k_hankel_pp, k_hankel_fast (STG/WarpSync, 1024/6144/8192), k_small,
k_hankel_1d, the four-step k_cols (PAIR/half), the 2D block plan and the
complex64 kernels.
"""

import numpy as np
import pytest
import torch

from oracle import hankel_oracle as O
from paper_1401_6238_b200 import batched

pytestmark = pytest.mark.gpu

CASES = [
    # (shape, batch, real, c64)
    ((1024,) * 4, 301, False, False),   # k_hankel_pp
    ((80,) * 3, 203, False, False),     # k_hankel_fast L=256, cp.async staging, warp groups
    ((300,) * 3, 97, False, False),     # k_hankel_fast L=1024
    ((2000,) * 3, 45, False, False),    # k_hankel_fast L=6144
    ((2700,) * 3, 33, True, False),     # k_hankel_fast L=8192, real operands
    ((250,) * 3, 70, False, False),     # k_hankel_1d L=768
    ((5000,) * 3, 3, True, False),      # four-step, packed real pair + Hermitian half
    ((5000,) * 3, 3, False, False),     # four-step complex
    ((1024,) * 4, 301, False, True),    # complex64 fast kernel
    ((250,) * 3, 70, False, True),      # complex64 generic kernel
]


def _inputs(shape, B, real, c64, seed):
    rng = np.random.default_rng(seed)
    d = sum(shape) - len(shape) + 1
    mk = (lambda *s: rng.standard_normal(s)) if real else \
        (lambda *s: rng.standard_normal(s) + 1j * rng.standard_normal(s))
    h, x = mk(B, d), mk(B, shape[1])
    if c64:
        h, x = h.astype(np.float32 if real else np.complex64), \
            x.astype(np.float32 if real else np.complex64)
    return torch.from_numpy(h).cuda(), torch.from_numpy(x).cuda()


def _run(dh, dx, shape, pad_rows=2):
    """Product into the middle of a NaN-poisoned buffer with guard rows."""
    B = dh.shape[0]
    dt = torch.complex64 if dh.dtype in (torch.complex64, torch.float32) else torch.complex128
    buf = torch.full((B + 2 * pad_rows, shape[0]), complex(float("nan"), float("nan")),
                     dtype=dt, device=dh.device)
    out = buf[pad_rows:pad_rows + B]
    batched.hankel_tvp_partial(dh, [dx] * (len(shape) - 1), shape, out=out)
    torch.cuda.synchronize()
    b = buf.cpu().numpy()
    assert np.isnan(b[:pad_rows]).all() and np.isnan(b[pad_rows + B:]).all(), "guard rows written"
    y = b[pad_rows:pad_rows + B]
    assert not np.isnan(y).any(), "output element left unwritten"
    return y


@pytest.mark.parametrize("shape,B,real,c64", CASES)
def test_items_bitwise_independent_of_batch_position(shape, B, real, c64, monkeypatch):
    # single-item sub-batches would otherwise go to the latency kernel (k_small),
    # a different arithmetic order; its own parity is covered elsewhere
    monkeypatch.setenv("HK_NO_SMALL", "1")
    dh, dx = _inputs(shape, B, real, c64, seed=B)
    full = _run(dh, dx, shape)
    again = _run(dh, dx, shape)
    assert np.array_equal(full, again), "repeated launch differs"
    # sub-batches at other offsets / sizes (tails, ping-pong and staging slots shift)
    for lo, hi in [(0, 1), (1, 2), (B // 3, B // 3 + B // 2), (B - 1, B), (1, B)]:
        if hi <= lo:
            continue
        sub = _run(dh[lo:hi].contiguous(), dx[lo:hi].contiguous(), shape)
        assert np.array_equal(sub, full[lo:hi]), f"items {lo}:{hi} differ by batch position"
    # and the values are right (oracle, first and last item)
    tol = 1e-4 if c64 else 1e-10
    for b in (0, B - 1):
        c = lambda a: a.cpu().numpy().astype(np.complex128)
        ref = O.hankel_tvp_partial(c(dh[b]), shape, [c(dx[b])] * (len(shape) - 1))
        assert np.linalg.norm(full[b] - ref) <= tol * np.linalg.norm(ref)


def test_block_plan_bitwise_independent_of_batch_position():
    rng = np.random.default_rng(5)
    B = 9
    H = rng.standard_normal((B, 118, 148)) + 1j * rng.standard_normal((B, 118, 148))
    X = rng.standard_normal((B, 40, 50)) + 1j * rng.standard_normal((B, 40, 50))
    dH = torch.from_numpy(H).cuda()
    dx = torch.from_numpy(np.ascontiguousarray(np.transpose(X, (0, 2, 1)))).cuda().reshape(B, -1)
    f = lambda a, b: batched.bhhb_tvp_partial(dH[a:b].contiguous(), [dx[a:b].contiguous()] * 2,
                                             3, (40,) * 3, (50,) * 3).cpu().numpy()
    full = f(0, B)
    assert np.array_equal(full, f(0, B))
    assert np.array_equal(full[3:7], f(3, 7))
    ref = O.bhhb_tvp_partial_batch(H[:1], X[:1], (40,) * 3, (50,) * 3)
    assert np.linalg.norm(full[0] - ref[0]) <= 1e-10 * np.linalg.norm(ref[0])

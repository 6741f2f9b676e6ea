"""Randomised parity sweep over every dispatch path (latency kernel, ping-pong,
fast, generic, two-level with packed/Hermitian real passes, block) against the
CPU oracle: seeded shapes, orders, dtypes, batch sizes and repeated vectors."""

import numpy as np
import pytest
import torch

from oracle import hankel_oracle as O
from paper_1401_6238_b200 import batched
from tests.helpers import strict_relerr

pytestmark = pytest.mark.gpu

TOL = 1e-10


def _vec(rng, shape, real):
    v = rng.standard_normal(shape)
    return v if real else v + 1j * rng.standard_normal(shape)


CASES = []
_rng = np.random.default_rng(2024)
for k in range(120):
    m = int(_rng.integers(2, 5))
    scale = [40, 400, 1400, 5000, 30000][k % 5]
    shape = tuple(int(_rng.integers(1, scale) + 1) for _ in range(m))
    if k % 3 == 0:  # H x^{m-1}: equal trailing modes, one repeated vector
        shape = (shape[0],) + (shape[1],) * (m - 1)
    if sum(shape) - m + 1 > 200_000:
        shape = tuple(max(1, n // 4) for n in shape)
    B = int(_rng.choice([1, 2, 5, 40, 200])) if sum(shape) < 20000 else int(_rng.choice([1, 2]))
    real = bool(_rng.integers(0, 2))
    same = bool(_rng.integers(0, 2))
    CASES.append((k, shape, B, real, same))


@pytest.mark.parametrize("k,shape,B,real,same", CASES)
def test_random_products(k, shape, B, real, same):
    rng = np.random.default_rng(1000 + k)
    m = len(shape)
    d = sum(shape) - m + 1
    h = _vec(rng, (B, d), real)
    if same and len(set(shape[1:])) == 1:
        x = _vec(rng, (B, shape[1]), real)
        xs_np = [x] * (m - 1)
        dx = torch.from_numpy(x).cuda()
        xs = [dx] * (m - 1)
    else:
        xs_np = [_vec(rng, (B, n), real) for n in shape[1:]]
        xs = [torch.from_numpy(x).cuda() for x in xs_np]
    y = batched.hankel_tvp_partial(torch.from_numpy(h).cuda(), xs, shape).cpu().numpy()
    for b in range(min(B, 3)):
        ref = O.hankel_tvp_partial(h[b], shape, [x[b] for x in xs_np])
        assert strict_relerr(y[b], ref) <= TOL, (k, shape, B, b)
    # full product with one more vector of mode-1 length
    x1 = _vec(rng, (B, shape[0]), real)
    a = batched.hankel_tvp_full(torch.from_numpy(h).cuda(), [torch.from_numpy(x1).cuda()] + xs,
                                shape).cpu().numpy()
    for b in range(min(B, 3)):
        a_ref = O.hankel_tvp_full(h[b], shape, [x1[b]] + [x[b] for x in xs_np])
        # alpha = x1 . (H x_2 .. x_m): bound the error by |x1| |y| (a sum that
        # cancels is not an error of the product)
        y_ref = O.hankel_tvp_partial(h[b], shape, [x[b] for x in xs_np])
        scale = np.linalg.norm(x1[b]) * np.linalg.norm(y_ref)
        assert abs(a[b] - a_ref) <= TOL * scale, (k, shape, B, b)


BLOCK_CASES = []
_rng2 = np.random.default_rng(77)
for k in range(30):
    m = int(_rng2.integers(2, 4))
    top = [12, 40, 90][k % 3]
    block = tuple(int(_rng2.integers(1, top) + 1) for _ in range(m))
    outer = tuple(int(_rng2.integers(1, top) + 1) for _ in range(m))
    if k % 2 == 0:  # repeated vector
        block = (block[0],) + (block[1],) * (m - 1)
        outer = (outer[0],) + (outer[1],) * (m - 1)
    B = int(_rng2.choice([1, 3, 17]))
    BLOCK_CASES.append((k, block, outer, B))


@pytest.mark.parametrize("k,block,outer,B", BLOCK_CASES)
def test_random_block_products(k, block, outer, B):
    rng = np.random.default_rng(5000 + k)
    m = len(block)
    din, dout = sum(block) - m + 1, sum(outer) - m + 1
    H = rng.standard_normal((B, din, dout)) + 1j * rng.standard_normal((B, din, dout))
    same = k % 2 == 0
    xs_np = []
    for p in range(1, m):
        if same and p > 1:
            xs_np.append(xs_np[0])
        else:
            n = block[p] * outer[p]
            xs_np.append(rng.standard_normal((B, n)) + 1j * rng.standard_normal((B, n)))
    dH = torch.from_numpy(H).cuda()
    dxs, seen = [], {}
    for x in xs_np:
        if id(x) not in seen:
            seen[id(x)] = torch.from_numpy(x).cuda()
        dxs.append(seen[id(x)])
    y = batched.bhhb_tvp_partial(dH, dxs, m, block, outer).cpu().numpy()
    for b in range(min(B, 3)):
        ref = O.bhhb_tvp_partial(H[b], block, outer, [x[b] for x in xs_np])
        assert strict_relerr(y[b], ref) <= TOL, (k, block, outer, B, b)


TM_CASES = []
_rng3 = np.random.default_rng(99)
for k in range(16):
    m = int(_rng3.integers(2, 4))
    n = int(_rng3.integers(2, 600))
    shape = (int(_rng3.integers(2, 600)),) + (n,) * (m - 1)
    r = int(_rng3.integers(1, 6))
    TM_CASES.append((k, shape, r, int(_rng3.choice([1, 3]))))


@pytest.mark.parametrize("k,shape,r,B", TM_CASES)
def test_random_times_matrices(k, shape, r, B):
    """times_matrices (hankel.py:174-194) with the same matrix for every mode
    (symmetric dedupe + mirrored stores) and with distinct matrices."""
    rng = np.random.default_rng(9000 + k)
    m = len(shape)
    d = sum(shape) - m + 1
    h = rng.standard_normal((B, d)) + 1j * rng.standard_normal((B, d))
    U = rng.standard_normal((B, shape[1], r)) + 1j * rng.standard_normal((B, shape[1], r))
    dU = torch.from_numpy(U).cuda()
    T = batched.times_matrices(torch.from_numpy(h).cuda(), shape, [dU] * (m - 1)).cpu().numpy()
    mats = [rng.standard_normal((B, shape[1], r)) + 1j * rng.standard_normal((B, shape[1], r))
            for _ in range(m - 1)]
    T2 = batched.times_matrices(torch.from_numpy(h).cuda(), shape,
                                [torch.from_numpy(M).cuda() for M in mats]).cpu().numpy()
    for b in range(B):
        ref = O.times_matrices(h[b], shape, [U[b]] * (m - 1))
        assert strict_relerr(T[b], ref) <= TOL, (k, shape, r, b)
        ref2 = O.times_matrices(h[b], shape, [M[b] for M in mats])
        assert strict_relerr(T2[b], ref2) <= TOL, (k, shape, r, b)

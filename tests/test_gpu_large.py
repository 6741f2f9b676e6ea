"""GPU parity of the two-level (large-L four-step and 2D block) kernels
against the CPU oracle and the reference golden outputs (cfg3, cfg4)."""

import numpy as np
import pytest
import torch

import paper_1401_6238_b200 as P
from oracle import hankel_oracle as O
from paper_1401_6238_b200 import batched, workloads
from tests.helpers import load_golden, rand_vec, strict_relerr

pytestmark = pytest.mark.gpu

TOL = 1e-10


@pytest.mark.parametrize("shape", [(3000, 3000, 3000), (5000, 4000), (20000, 9000, 30),
                                   (4096, 4096, 4096, 4096)])
def test_large_1d_partial_and_full(shape):
    rng = np.random.default_rng(sum(shape))
    d = sum(shape) - len(shape) + 1
    h = rand_vec(rng, d)
    xs = [rand_vec(rng, n) for n in shape]
    H = P.HankelTensor(shape, h)
    y = H.tvp_partial(xs[1:])
    ref = O.hankel_tvp_partial(h, shape, xs[1:])
    assert strict_relerr(y, ref) <= TOL
    a = H.tvp_full(xs)
    a_ref = O.hankel_tvp_full(h, shape, xs)
    assert abs(a - a_ref) <= TOL * abs(a_ref)


def test_large_1d_batched_mixed_real():
    rng = np.random.default_rng(5)
    shape = (4000, 3000, 2000)
    d = sum(shape) - 2
    B = 3
    h = rng.standard_normal((B, d))
    x2 = rng.standard_normal((B, shape[1]))
    x3 = rng.standard_normal((B, shape[2])) + 1j * rng.standard_normal((B, shape[2]))
    y = batched.hankel_tvp_partial(torch.from_numpy(h).cuda(),
                                   [torch.from_numpy(x2).cuda(), torch.from_numpy(x3).cuda()],
                                   shape).cpu().numpy()
    ref = np.stack([O.hankel_tvp_partial(h[b], shape, [x2[b], x3[b]]) for b in range(B)])
    assert strict_relerr(y, ref) <= TOL
    spec = batched.hankel_spectrum(torch.from_numpy(h).cuda(), shape)
    y2 = batched.hankel_tvp_partial(spec, [torch.from_numpy(x2).cuda(),
                                           torch.from_numpy(x3).cuda()], shape,
                                    spectrum=True).cpu().numpy()
    assert strict_relerr(y2, ref) <= TOL


@pytest.mark.parametrize("block,outer", [((40, 40, 40), (40, 40, 40)),
                                         ((30, 50, 20), (25, 40, 30)),
                                         ((60, 70), (70, 60)),
                                         # unequal modes / cfg4 shape: caught a reduction
                                         # race between warp-synchronous row groups
                                         ((60, 70), (60, 70)),
                                         ((50, 80), (64, 64)),
                                         ((64, 64, 64), (64, 64, 64))])
def test_block_two_level_vs_oracle(block, outer):
    rng = np.random.default_rng(len(block) * 7 + block[0])
    m = len(block)
    din, dout = sum(block) - m + 1, sum(outer) - m + 1
    Hm = rand_vec(rng, din * dout).reshape(din, dout)
    T = P.BhhbTensor(m, block, outer, Hm)
    assert T._two_level
    xs = [rand_vec(rng, n * N) for n, N in zip(block, outer)]
    assert strict_relerr(T.tvp_partial(xs[1:]), O.bhhb_tvp_partial(Hm, block, outer, xs[1:])) <= TOL
    a_ref = O.bhhb_tvp_full(Hm, block, outer, xs)
    assert abs(T.tvp_full(xs) - a_ref) <= TOL * abs(a_ref)


def test_cfg4_batch_vs_golden():
    g = load_golden("cfg4.npz")
    H, X = workloads.cfg4()
    H, X = H[:64], X[:64]
    dH = torch.from_numpy(np.ascontiguousarray(H)).cuda()
    dx = torch.from_numpy(np.ascontiguousarray(np.transpose(X, (0, 2, 1)))).cuda().reshape(64, -1)
    y = batched.bhhb_tvp_partial(dH, [dx, dx], 3, (64,) * 3, (64,) * 3).cpu().numpy()
    assert strict_relerr(y[0], g["y"][0]) <= TOL
    np.testing.assert_allclose(np.linalg.norm(y, axis=1), g["norms"][:64], rtol=TOL)
    ref = O.bhhb_tvp_partial_batch(H[:8], X[:8], (64,) * 3, (64,) * 3)
    assert strict_relerr(y[:8], ref) <= TOL


def test_cfg3_vs_golden():
    g = load_golden("cfg3.npz")
    h, x = workloads.cfg3()
    dh = torch.from_numpy(h).cuda()[None]
    dx = torch.from_numpy(x).cuda()[None]
    y = batched.hankel_tvp_partial(dh, [dx, dx], (1 << 22,) * 3)[0].cpu().numpy()
    assert strict_relerr(y[g["idx"]], g["y"]) <= TOL
    assert abs(np.linalg.norm(y) - float(g["norm"])) <= TOL * float(g["norm"])


@pytest.mark.parametrize("L1", [8, 12, 16, 24, 32, 48, 64, 96, 128, 192, 256, 384, 512, 768,
                                1024, 1536, 2048])
def test_every_column_length(L1):
    """Two-level 1D plans forced onto each column length (fft_len = L1 * 4096)."""
    rng = np.random.default_rng(L1)
    L = L1 * 4096
    n = (L - 1) // 2 + 1            # order-2 tensor with d_H <= L and > 8192
    shape = (n // 3, L - n // 3 - 1)
    shape = (max(1, shape[0]), max(1, min(shape[1], L // 2)))
    d = sum(shape) - 1
    h = rand_vec(rng, d)
    x = rand_vec(rng, shape[1])
    dh = torch.from_numpy(h).cuda()[None]
    dx = torch.from_numpy(x).cuda()[None]
    y = batched.hankel_tvp_partial(dh, [dx], shape, fft_len=L)[0].cpu().numpy()
    ref = O.hankel_tvp_partial(h, shape, [x])
    assert strict_relerr(y, ref) <= TOL


@pytest.mark.parametrize("L1", [8, 12, 48, 96, 192, 384, 768, 1536])
def test_real_pair_column_pass(L1):
    """Real h with ONE real vector takes the packed z = h + i x column pass
    (ST_A_PAIR): partial and full products, batch 2, forced column length."""
    rng = np.random.default_rng(100 + L1)
    L = L1 * 4096
    n = L // 3                       # order 3: d_H = 3n - 2 <= L, two-level (> 8192)
    shape = (n, n, n)
    B = 2
    h = rng.standard_normal((B, 3 * n - 2))
    x = rng.uniform(-1.0, 1.0, (B, n))
    dh = torch.from_numpy(h).cuda()
    dx = torch.from_numpy(x).cuda()
    y = batched.hankel_tvp_partial(dh, [dx, dx], shape, fft_len=L).cpu().numpy()
    a = batched.hankel_tvp_full(dh, [dx, dx, dx], shape, fft_len=L).cpu().numpy()
    for b in range(B):
        ref = O.hankel_tvp_partial(h[b], shape, [x[b], x[b]])
        assert strict_relerr(y[b], ref) <= TOL
        a_ref = O.hankel_tvp_full(h[b], shape, [x[b]] * 3)
        assert abs(a[b] - a_ref) <= TOL * abs(a_ref)


@pytest.mark.parametrize("shape", [
    # x rows (n / 4096) below one 256-row block: no 4-D block copy for x, one partial box
    (7_500_000, 500_000, 500_000),
    # x rows an exact multiple of 256 (512 rows, no partial row, no partial block)
    (5_000_000, 1 << 21, 1 << 21),
    # partial last row inside a partial block for both operands
    (4_500_000, 2_000_000, 2_000_000),
])
def test_packed_real_tma_column_blocks(shape):
    """Real h and one real vector at L = 3072 x 4096 (packed TMA column pass,
    Hermitian half): operand row counts around the 256-row block edges of the
    4-D / 3-D tensor copies (reference hankel.py:140-147, padded oracle)."""
    rng = np.random.default_rng(shape[1] % 1000)
    d = sum(shape) - 2
    assert (1 << 23) < d <= 3 * (1 << 22)
    h = rng.standard_normal(d)
    x = rng.uniform(-1.0, 1.0, shape[1])
    y = batched.hankel_tvp_partial(torch.from_numpy(h).cuda()[None],
                                   [torch.from_numpy(x).cuda()[None]] * 2, shape)[0].cpu().numpy()
    ref = O.hankel_tvp_partial_padded(h, shape, [x, x], length=1 << 24)
    assert strict_relerr(y, ref) <= TOL

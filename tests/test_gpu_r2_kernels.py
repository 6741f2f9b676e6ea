"""GPU parity of the round-2 kernel variants against the oracle / reference
goldens: the TMA column kernel (both column lengths, complex and real
operands, strided items), the ping-pong row stage, the fused BHHB kernel
(opt-in), and each A/B switch of the cfg2 kernel.  The library reads its HK_*
switches at every launch, so one process exercises every variant."""

import numpy as np
import pytest
import torch

import paper_1401_6238_b200 as P
from oracle import hankel_oracle as O
from paper_1401_6238_b200 import batched, workloads
from tests.helpers import load_golden, rand_vec, strict_relerr

pytestmark = pytest.mark.gpu

TOL = 1e-10


@pytest.mark.parametrize("env", [{}, {"HK_NO_COLTMA": "1"}, {"HK_COLTMA_STORE": "1"},
                                 {"HK_NO_PP_ROWS": "1"}, {"HK_PP_ROWS_TWO": "1"},
                                 {"HK_COL_NATSWZ": "0"}])
@pytest.mark.parametrize("shape,real", [((4200, 4200, 4200), True),      # L1 = 3072 x 4096
                                        ((4200, 4200, 4200), False),
                                        ((2100, 2100, 2100), True),      # 1536 x 4096
                                        ((9000, 9000), False)])
def test_four_step_variants(monkeypatch, env, shape, real):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    rng = np.random.default_rng(sum(shape) + real)
    d = sum(shape) - len(shape) + 1
    if real:
        h = rng.standard_normal(d)
        xs = [rng.standard_normal(n) for n in shape]
    else:
        h = rand_vec(rng, d)
        xs = [rand_vec(rng, n) for n in shape]
    H = P.HankelTensor(shape, h)
    ref = O.hankel_tvp_partial(h, shape, xs[1:])
    assert strict_relerr(H.tvp_partial(xs[1:]), ref) <= TOL


def test_four_step_batch_item_strides(monkeypatch):
    """Several items per call: the TMA maps carry the item stride."""
    shape = (3000, 3000, 3000)
    d = sum(shape) - 2
    rng = np.random.default_rng(5)
    B = 3
    h = rng.standard_normal((B, d))
    x = rng.standard_normal((B, shape[1]))
    dh = torch.from_numpy(h).cuda()
    dx = torch.from_numpy(x).cuda()
    y = batched.hankel_tvp_partial(dh, [dx, dx], shape).cpu().numpy()
    for b in range(B):
        ref = O.hankel_tvp_partial(h[b], shape, [x[b], x[b]])
        assert strict_relerr(y[b], ref) <= TOL


def test_cfg3_golden_every_row_variant(monkeypatch):
    g = load_golden("cfg3.npz")
    h, x = workloads.cfg3()
    dh = torch.from_numpy(h).cuda()[None]
    dx = torch.from_numpy(x).cuda()[None]
    for env in ({}, {"HK_NO_PP_ROWS": "1"}, {"HK_NO_COLTMA": "1"}):
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        y = batched.hankel_tvp_partial(dh, [dx, dx], (1 << 22,) * 3)[0].cpu().numpy()
        assert strict_relerr(y[g["idx"]], g["y"]) <= TOL
        for k in env:
            monkeypatch.delenv(k)


@pytest.mark.parametrize("block,outer", [((64, 64, 64), (64, 64, 64)), ((40, 40, 40), (64, 64, 64)),
                                         ((64, 64, 64), (20, 20, 20)), ((33, 33), (64, 64)),
                                         ((50, 64, 64), (30, 64, 64))])
def test_bhhb_fused_vs_oracle(monkeypatch, block, outer):
    monkeypatch.setenv("HK_BHHB_FUSED", "1")
    rng = np.random.default_rng(sum(block) + 3 * sum(outer))
    m = len(block)
    din, dout = sum(block) - m + 1, sum(outer) - m + 1
    Hm = rand_vec(rng, din * dout).reshape(din, dout)
    T = P.BhhbTensor(m, block, outer, Hm)
    x = rand_vec(rng, block[1] * outer[1])
    xs = [x] * (m - 1) if len(set(block[1:])) == 1 and len(set(outer[1:])) == 1 else None
    if xs is None:
        pytest.skip("the fused kernel covers one distinct vector")
    ref = O.bhhb_tvp_partial(Hm, block, outer, xs)
    assert strict_relerr(T.tvp_partial(xs), ref) <= TOL


def test_bhhb_fused_cfg4_golden(monkeypatch):
    monkeypatch.setenv("HK_BHHB_FUSED", "1")
    g = load_golden("cfg4.npz")
    H, X = workloads.cfg4()
    H, X = H[:160], X[:160]     # > one item per CTA on a 148-SM part
    dH = torch.from_numpy(np.ascontiguousarray(H)).cuda()
    dx = torch.from_numpy(np.ascontiguousarray(np.transpose(X, (0, 2, 1)))).cuda().reshape(160, -1)
    y = batched.bhhb_tvp_partial(dH, [dx, dx], 3, (64,) * 3, (64,) * 3).cpu().numpy()
    assert strict_relerr(y[0], g["y"][0]) <= TOL
    np.testing.assert_allclose(np.linalg.norm(y, axis=1), g["norms"][:160], rtol=TOL)


@pytest.mark.parametrize("twv", ["2", "8", "24", "56", "152"])
def test_cfg2_kernel_variants(monkeypatch, twv):
    monkeypatch.setenv("HK_PP_TWV", twv)
    g = load_golden("cfg2.npz")
    h, x = workloads.cfg2()
    B = 300
    dh = torch.from_numpy(h[:B]).cuda()
    dx = torch.from_numpy(x[:B]).cuda()
    y = batched.hankel_tvp_partial(dh, [dx, dx, dx], (1024,) * 4).cpu().numpy()
    np.testing.assert_allclose(np.linalg.norm(y, axis=1), g["norms"][:B], rtol=TOL)
    ref = O.hankel_tvp_partial(h[0], (1024,) * 4, [x[0]] * 3)
    assert strict_relerr(y[0], ref) <= TOL


@pytest.mark.parametrize("block,outer,B", [((64, 64, 64), (20, 20, 20), 3),   # 64-point columns
                                           ((60, 60, 60), (64, 64, 64), 2),
                                           ((64, 64), (50, 50), 5),
                                           ((32, 32, 32), (40, 40, 40), 3)])  # 96-point rows
def test_block_rows_pp256_vs_fast_rows(monkeypatch, block, outer, B):
    """The 256-point row kernel (units of 16 rows, several items per launch)
    against the fast-kernel row stage and the oracle."""
    rng = np.random.default_rng(sum(block) * 3 + sum(outer) + B)
    m = len(block)
    din, dout = sum(block) - m + 1, sum(outer) - m + 1
    H = rand_vec(rng, B * din * dout).reshape(B, din, dout)
    X = rand_vec(rng, B * block[1] * outer[1]).reshape(B, outer[1], block[1])  # (B, N, n)
    dH = torch.from_numpy(H).cuda()
    dx = torch.from_numpy(np.ascontiguousarray(X)).cuda().reshape(B, -1)
    xs = [dx] * (m - 1)
    y = batched.bhhb_tvp_partial(dH, xs, m, block, outer).cpu().numpy()
    monkeypatch.setenv("HK_NO_PP256", "1")
    y2 = batched.bhhb_tvp_partial(dH, xs, m, block, outer).cpu().numpy()
    assert strict_relerr(y, y2) <= 1e-13
    for b in range(B):
        xv = X[b].reshape(-1)
        ref = O.bhhb_tvp_partial(H[b], block, outer, [xv] * (m - 1))
        assert strict_relerr(y[b], ref) <= TOL


@pytest.mark.parametrize("block,outer,B", [((62, 62, 62), (28, 28, 28), 3),
                                           ((64, 64, 64), (63, 63, 63), 2)])
def test_block_rows_pp192_opt_in(monkeypatch, block, outer, B):
    """HK_PP192=1 (read when the plan is created: shapes no other test uses):
    the row stage at the exact padded length 192 = 16 x 12 on the ping-pong row
    kernel, 16 threads per product with 12 live in the radix-16 pass, against
    the oracle (reference block.py:136-144)."""
    monkeypatch.setenv("HK_PP192", "1")
    rng = np.random.default_rng(sum(block) + 7 * sum(outer) + B)
    m = len(block)
    din, dout = sum(block) - m + 1, sum(outer) - m + 1
    assert 128 < din <= 192
    H = rand_vec(rng, B * din * dout).reshape(B, din, dout)
    X = rand_vec(rng, B * block[1] * outer[1]).reshape(B, outer[1], block[1])  # (B, N, n)
    dH = torch.from_numpy(H).cuda()
    dx = torch.from_numpy(np.ascontiguousarray(X)).cuda().reshape(B, -1)
    y = batched.bhhb_tvp_partial(dH, [dx] * (m - 1), m, block, outer).cpu().numpy()
    for b in range(B):
        ref = O.bhhb_tvp_partial(H[b], block, outer, [X[b].reshape(-1)] * (m - 1))
        assert strict_relerr(y[b], ref) <= TOL

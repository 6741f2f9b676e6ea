"""complex64 / float32 variant (north_star: relative error <= 1e-4 for
fp32/complex64) against the oracle evaluated in complex128 on the same
(single-precision-rounded) inputs.  Reference algorithm: hankel.py:140-154."""

import numpy as np
import pytest
import torch

from oracle import hankel_oracle as O
from paper_1401_6238_b200 import batched, workloads
from tests.helpers import strict_relerr

pytestmark = pytest.mark.gpu

TOL = 1e-4


def _c64(a):
    return np.asarray(a).astype(np.complex64)


def test_cfg2_shape_c64_matches_oracle():
    h, x = workloads.cfg2()
    h, x = _c64(h[:96]), _c64(x[:96])
    dh, dx = torch.from_numpy(h).cuda(), torch.from_numpy(x).cuda()
    y = batched.hankel_tvp_partial(dh, [dx, dx, dx], (1024,) * 4)
    assert y.dtype == torch.complex64
    y = y.cpu().numpy()
    ref = O.hankel_tvp_partial_batch(h.astype(np.complex128), [x.astype(np.complex128)] * 3,
                                     (1024,) * 4)
    err = strict_relerr(y, ref)
    assert err <= TOL, err
    # FP32 arithmetic really ran (not a complex128 path rounded at the end)
    assert err > 1e-9


@pytest.mark.parametrize("shape", [(5, 6), (40, 33, 7), (100,) * 3, (300, 200, 120),
                                   (700, 800), (1000, 1000, 900), (2000, 2000, 2000),
                                   (2047, 2048, 2048, 2048), (3, 4, 2, 5)])
def test_c64_partial_and_full_lengths(shape):
    rng = np.random.default_rng(sum(shape))
    B = 7
    d = sum(shape) - len(shape) + 1
    h = _c64(rng.standard_normal((B, d)) + 1j * rng.standard_normal((B, d)))
    xs = [_c64(rng.standard_normal((B, n)) + 1j * rng.standard_normal((B, n))) for n in shape]
    dh = torch.from_numpy(h).cuda()
    dxs = [torch.from_numpy(x).cuda() for x in xs]
    y = batched.hankel_tvp_partial(dh, dxs[1:], shape).cpu().numpy()
    a = batched.hankel_tvp_full(dh, dxs, shape).cpu().numpy()
    c = lambda v: v.astype(np.complex128)
    for b in range(B):
        ref = O.hankel_tvp_partial(c(h[b]), shape, [c(x[b]) for x in xs[1:]])
        assert strict_relerr(y[b], ref) <= TOL
        refa = O.hankel_tvp_full(c(h[b]), shape, [c(x[b]) for x in xs])
        yb = O.hankel_tvp_partial(c(h[b]), shape, [c(x[b]) for x in xs[1:]])
        # a full product may cancel: bound by ||x_1|| ||H x_2..x_m||
        assert abs(a[b] - refa) <= TOL * np.linalg.norm(xs[0][b]) * np.linalg.norm(yb)


def test_c64_real_float32_inputs():
    h, x = workloads.cfg1()
    dh = torch.from_numpy(h.astype(np.float32)).cuda()[None]
    dx = torch.from_numpy(x.astype(np.float32)).cuda()[None]
    y = batched.hankel_tvp_partial(dh, [dx, dx], (100,) * 3)[0].cpu().numpy()
    ref = O.hankel_tvp_partial(h.astype(np.float32).astype(np.float64), (100,) * 3,
                               [x.astype(np.float32).astype(np.float64)] * 2)
    assert strict_relerr(y, ref) <= TOL


def test_c64_mixed_precision_and_two_level_rejected():
    h = torch.zeros((2, 298), dtype=torch.complex64, device="cuda")
    x = torch.zeros((2, 100), dtype=torch.complex128, device="cuda")
    with pytest.raises(ValueError):
        batched.hankel_tvp_partial(h, [x, x], (100,) * 3)
    hb = torch.zeros((1, 3 * 2999 + 1), dtype=torch.complex64, device="cuda")
    xb = torch.zeros((1, 3000), dtype=torch.complex64, device="cuda")
    with pytest.raises(NotImplementedError):
        batched.hankel_tvp_partial(hb, [xb, xb], (3000,) * 3)


@pytest.mark.parametrize("shape,B", [((1024,) * 4, 1), ((1024,) * 4, 151), ((1024,) * 4, 299),
                                     ((1000, 1024, 1024, 1024), 5),   # even d_H: 16-byte rows
                                     ((800,) * 5, 3), ((1024, 1024, 1024), 150),
                                     ((1024, 700, 700), 8), ((333, 777, 777, 777), 4)])
def test_c64_pingpong_kernel_shapes(shape, B, monkeypatch):
    """The complex64 ping-pong kernel (one repeated vector, L = 4096, x and y
    within the first quarter): batch sizes around the grid size (tails of one
    and two groups), odd and even generator lengths, orders 3-5; and the same
    launch on the fast kernel (HK_NO_PP_C64=1) as a cross-check."""
    rng = np.random.default_rng(sum(shape) + B)
    d = sum(shape) - len(shape) + 1
    assert 2048 < d <= 4096 and max(shape[1:]) <= 1024 and shape[0] <= 1024
    h = _c64(rng.standard_normal((B, d)) + 1j * rng.standard_normal((B, d)))
    x = _c64(rng.standard_normal((B, shape[1])) + 1j * rng.standard_normal((B, shape[1])))
    dh, dx = torch.from_numpy(h).cuda(), torch.from_numpy(x).cuda()
    y = batched.hankel_tvp_partial(dh, [dx] * (len(shape) - 1), shape).cpu().numpy()
    monkeypatch.setenv("HK_NO_PP_C64", "1")
    y2 = batched.hankel_tvp_partial(dh, [dx] * (len(shape) - 1), shape).cpu().numpy()
    assert strict_relerr(y, y2) <= 1e-5
    c = lambda v: v.astype(np.complex128)
    for b in sorted({0, B // 2, B - 1}):
        ref = O.hankel_tvp_partial(c(h[b]), shape, [c(x[b])] * (len(shape) - 1))
        assert strict_relerr(y[b], ref) <= TOL

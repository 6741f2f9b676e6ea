"""Round-2 parity cases against the REFERENCE's own outputs
(oracle/gen_golden_r2.py):

* times_matrices / HOOI on two-level plans (d_H > 8192), reference
  hankel.py:174-194 -- order 3 n=3000 r=3 (same and distinct matrices) and
  order 2 (5000, 4000) r=2;
* the cfg5 loop after 50 sweeps (final-U projector);
* hooi_symmetric on rank-deficient Hankel and on BHHB tensors
  (decompose.py:142-184 accepts any square structured tensor);
* BHHB generators outside the native 2D plan fall back to the Kronecker-1D
  form instead of failing.
"""

import numpy as np
import pytest
import torch

import paper_1401_6238_b200 as P
from oracle import hankel_oracle as O
from paper_1401_6238_b200 import batched, workloads
from paper_1401_6238_b200.hooi import hooi_symmetric, hooi_symmetric_batched
from tests.helpers import load_golden, rand_vec, strict_relerr

pytestmark = pytest.mark.gpu


def _proj_err(U, Uref):
    P1, P2 = U @ U.conj().T, Uref @ Uref.conj().T
    return np.linalg.norm(P1 - P2) / np.linalg.norm(P2)


def test_times_matrices_two_level_order3_same_and_mixed():
    g = load_golden("tm_large.npz")
    h3, M, M2, _, _ = workloads.tm_large_inputs()
    H = P.HankelTensor((3000,) * 3, h3)
    assert strict_relerr(H.times_matrices([M, M]), g["T3_same"]) <= 1e-10
    assert strict_relerr(P.times_matrices(H, [M, M2]), g["T3_mixed"]) <= 1e-10


def test_times_matrices_two_level_order2():
    g = load_golden("tm_large.npz")
    _, _, _, h2, Mb = workloads.tm_large_inputs()
    H = P.HankelTensor((5000, 4000), h2)
    assert strict_relerr(H.times_matrices([Mb]), g["T2"]) <= 1e-10


def test_times_matrices_two_level_batched_raw_h_and_spectrum():
    """Batched engine, raw h and cached spectrum, several items, rank 1..3."""
    g = load_golden("tm_large.npz")
    h3, M, M2, _, _ = workloads.tm_large_inputs()
    shape = (3000,) * 3
    dh = torch.from_numpy(np.stack([h3, 2 * h3])).cuda()
    dM = torch.from_numpy(np.stack([M, M])).cuda()
    T = batched.times_matrices(dh, shape, [dM, dM]).cpu().numpy()
    assert strict_relerr(T[0], g["T3_same"]) <= 1e-10
    assert strict_relerr(T[1], 2 * g["T3_same"]) <= 1e-10
    spec = batched.hankel_spectrum(dh, shape)
    dM2 = torch.from_numpy(np.stack([M2, M2])).cuda()
    T = batched.times_matrices(spec, shape, [dM, dM2], spectrum=True).cpu().numpy()
    assert strict_relerr(T[0], g["T3_mixed"]) <= 1e-10
    # rank-1 column slice of the same case
    T1 = batched.times_matrices(dh[:1], shape, [dM[:1, :, :1].contiguous()] * 2)
    assert strict_relerr(T1[0].cpu().numpy()[:, 0, 0], g["T3_same"][:, 0, 0]) <= 1e-10


def test_hooi_two_level_shape_runs_and_matches_oracle_products():
    """hooi_symmetric on an order-3 n=3000 Hankel tensor (d_H = 8998 > 8192)."""
    h3 = workloads.tm_large_inputs()[0]
    H = P.HankelTensor((3000,) * 3, h3)
    res = hooi_symmetric(H, 2, max_iter=2)
    U = res.factor
    assert np.abs(U.conj().T @ U - np.eye(2)).max() <= 1e-10
    # the core matches the oracle's products with the returned factor
    T = O.times_matrices_fast(h3, (3000,) * 3, [np.conj(U)] * 2)
    S = np.moveaxis(np.tensordot(T, np.conj(U), axes=([0], [0])), -1, 0)
    assert strict_relerr(res.core, S) <= 1e-10


def test_cfg5_fifty_sweeps_final_projector_matches_reference():
    g = load_golden("cfg5_sweep50.npz")
    sig, U0, shape = workloads.cfg5(signals=2)
    dh = torch.from_numpy(sig).cuda()
    U = hooi_symmetric_batched(dh, shape, 5, torch.from_numpy(U0).cuda(), max_iter=50)
    U = U.cpu().numpy()
    for s in range(2):
        assert _proj_err(U[s], g[f"U50_{s}"]) <= 1e-10


@pytest.mark.parametrize("name", ["rand", "rand4"])
def test_hooi_symmetric_hankel_matches_reference(name):
    g = load_golden("hooi_small.npz")
    h = g[f"{name}_h"]
    m = 3 if name == "rand" else 4
    n = (len(h) + m - 1) // m
    res = hooi_symmetric(P.HankelTensor((n,) * m, h), g[f"{name}_U"].shape[1], max_iter=30)
    assert _proj_err(res.factor, g[f"{name}_U"]) <= 1e-8
    assert abs(res.fits[-1] - g[f"{name}_fits"][-1]) <= 1e-10 * g[f"{name}_fits"][-1]
    assert np.abs(res.factor.conj().T @ res.factor - np.eye(res.factor.shape[1])).max() <= 1e-10


def test_hooi_symmetric_rank_deficient_factors_orthonormal():
    """All-ones tensor: rank-1 unfolding asked for rank 2."""
    g = load_golden("hooi_small.npz")
    res = hooi_symmetric(P.HankelTensor((5, 5, 5), np.ones(13)), 2)
    U = res.factor
    assert np.abs(U.conj().T @ U - np.eye(2)).max() <= 1e-10
    # the dominant direction and the fit are determined; the second column is not
    assert np.linalg.norm(U[:, 0] - g["ones_U"][:, 0]) <= 1e-10
    assert abs(res.fits[-1] - g["ones_fits"][-1]) <= 1e-10 * g["ones_fits"][-1]


def test_hooi_symmetric_accepts_bhhb():
    g = load_golden("hooi_small.npz")
    T = P.BhhbTensor(3, (2, 2, 2), (3, 3, 3), g["bhhb_H"])
    res = hooi_symmetric(T, 2, max_iter=30)
    assert _proj_err(res.factor, g["bhhb_U"]) <= 1e-8
    assert abs(res.fits[-1] - g["bhhb_fits"][-1]) <= 1e-10 * g["bhhb_fits"][-1]


def test_bhhb_times_matrices_native_two_level():
    """2D block plan (d_in*d_out > 8192): fused times_matrices vs the oracle loop."""
    rng = np.random.default_rng(91)
    block, outer = (40, 40, 40), (50, 50, 50)
    din, dout = 118, 148
    Hg = rand_vec(rng, din * dout).reshape(din, dout)
    T = P.BhhbTensor(3, block, outer, Hg)
    assert T._two_level
    M = rand_vec(rng, 2000 * 2).reshape(2000, 2)
    M2 = rand_vec(rng, 2000 * 3).reshape(2000, 3)
    for mats in ([M, M], [M, M2]):
        got = T.times_matrices(mats)
        ref = np.empty((2000, mats[0].shape[1], mats[1].shape[1]), dtype=np.complex128)
        for a in range(mats[0].shape[1]):
            for b in range(mats[1].shape[1]):
                ref[:, a, b] = O.bhhb_tvp_partial(Hg, block, outer,
                                                  [mats[0][:, a], mats[1][:, b]])
        assert strict_relerr(got, ref) <= 1e-10


def test_bhhb_outside_native_plan_falls_back_to_kronecker():
    """d_out = 4498 > 2048 (no 2D column plan): Kronecker-1D four-step instead."""
    rng = np.random.default_rng(92)
    block, outer = (2, 2, 2), (1500, 1500, 1500)
    Hg = rand_vec(rng, 4 * 4498).reshape(4, 4498)
    T = P.BhhbTensor(3, block, outer, Hg)
    assert not T._two_level
    x = rand_vec(rng, 3000)
    y = T.tvp_partial([x, x])
    assert strict_relerr(y, O.bhhb_tvp_partial(Hg, block, outer, [x, x])) <= 1e-10


def test_multi_device_sharded_product_matches_golden():
    """hankel_tvp_partial_multi: contiguous shards per device entry (the single
    GPU listed twice exercises the sharding/placement logic), host inputs."""
    g = load_golden("cfg2.npz")
    h, x = workloads.cfg2()
    hp = torch.from_numpy(h[:64]).pin_memory()
    xp = torch.from_numpy(x[:64]).pin_memory()
    outs = batched.hankel_tvp_partial_multi(hp, [xp, xp, xp], (1024,) * 4, devices=[0, 0, 0])
    assert [o.shape[0] for o in outs] == [22, 21, 21]
    y = batched.hankel_tvp_partial_multi(hp, [xp, xp, xp], (1024,) * 4, devices=[0, 0],
                                         gather_to=0).cpu().numpy()
    assert np.allclose(np.concatenate([o.cpu().numpy() for o in outs]), y, rtol=0, atol=0)
    for k, s in enumerate(g["sel"][:3]):
        assert strict_relerr(y[s], g["y"][k]) <= 1e-10
    norms = np.linalg.norm(y, axis=1)
    assert np.max(np.abs(norms - g["norms"][:64]) / g["norms"][:64]) <= 1e-10


@pytest.mark.parametrize("shape,real", [((10_000_000, 8_000_000), False),
                                        ((6_000_000,) * 3, True)])
def test_lengths_beyond_2_24(shape, real):
    """d_H ~ 1.8e7 > 2^24: four-step with a 3072-row column plan (L = 3072 x 8192)."""
    rng = np.random.default_rng(24)
    d = sum(shape) - len(shape) + 1
    mk = (lambda n: rng.standard_normal(n)) if real else (lambda n: rand_vec(rng, n))
    h = mk(d)
    xs = [mk(n) for n in shape[1:]]
    dh = torch.from_numpy(h).cuda()[None]
    dxs = [torch.from_numpy(x).cuda()[None] for x in xs]
    if len(xs) == 2:
        dxs = [dxs[0], dxs[0]]
        xs = [xs[0], xs[0]]
    y = batched.hankel_tvp_partial(dh, dxs, shape)[0].cpu().numpy()
    ref = O.hankel_tvp_partial_padded(h, shape, xs)
    assert strict_relerr(y, ref) <= 1e-10

"""GPU parity: the CUDA path (through the C ABI) against the reference's own
numbers (golden fixtures) and the pinned CPU oracle.

Tolerances (BASELINE.json north_star): relative error <= 1e-10 for
complex128/float64.  Small cases additionally meet the reference tests'
1e-11 bound (tests/test_hankel.py:136-145 et al.).
"""

import numpy as np
import pytest
import torch

import paper_1401_6238_b200 as P
from oracle import hankel_oracle as O
from paper_1401_6238_b200 import batched, workloads
from tests.helpers import load_golden, load_small_cases, rand_vec, relerr, strict_relerr

pytestmark = pytest.mark.gpu

TOL = 1e-10


@pytest.fixture(scope="module")
def small():
    return load_small_cases()


# ---- known answers ----------------------------------------------------------

def test_counting_example():
    H = P.HankelTensor((3, 3, 3), np.arange(7))
    np.testing.assert_allclose(H.tvp_partial([np.ones(3), np.ones(3)]), [18, 27, 36], atol=1e-11)


def test_zero_generator_and_zero_vector():
    H = P.HankelTensor((3, 3, 3), np.zeros(7))
    np.testing.assert_allclose(H.tvp_partial([np.ones(3)] * 2), 0, atol=1e-14)
    rng = np.random.default_rng(2)
    C = P.AntiCirculantTensor(3, 5, rand_vec(rng, 5))
    np.testing.assert_allclose(C.tvp_partial([np.zeros(5), rand_vec(rng, 5)]), 0, atol=1e-14)


def test_acirc_known_answers():
    C = P.AntiCirculantTensor(3, 3, [1, 2, 3])
    assert C.tvp_full([np.ones(3)] * 3) == pytest.approx(54.0)
    np.testing.assert_allclose(C.tvp_partial([np.ones(3)] * 2), 18 * np.ones(3), atol=1e-12)
    np.testing.assert_allclose(P.AntiCirculantTensor(3, 5, np.eye(5)[0]).spectrum,
                               np.full(5, 0.2), atol=1e-14)
    np.testing.assert_allclose(P.AntiCirculantTensor(2, 4, np.ones(4)).spectrum,
                               [1, 0, 0, 0], atol=1e-14)


def test_eigenpairs_random():
    # acceptance criterion 4 (tests/test_acceptance.py:112-124)
    rng = np.random.default_rng(104)
    for _ in range(50):
        m = int(rng.integers(2, 5))
        n = int(rng.integers(2, 9))
        C = P.AntiCirculantTensor(m, n, rand_vec(rng, n))
        for lam, v in C.special_eigenpairs():
            y = C.tvp_partial([v] * (m - 1))
            assert np.max(np.abs(y - lam * v)) <= 1e-10 * (1 + abs(lam))


# ---- reference golden small cases ------------------------------------------

def test_hankel_small_vs_reference(small):
    for shape, h, xs, y_ref, a_ref in small["hankel"]:
        H = P.HankelTensor(shape, h)
        if len(shape) < 2:
            continue
        assert strict_relerr(H.tvp_partial(xs[1:]), y_ref) <= 1e-12, shape
        assert abs(H.tvp_full(xs) - a_ref) <= 1e-12 * (1 + abs(a_ref)), shape


def test_acirc_small_vs_reference(small):
    for m, c, xs, spec_ref, y_ref, a_ref in small["acirc"]:
        A = P.AntiCirculantTensor(m, len(c), c)
        assert strict_relerr(A.spectrum, spec_ref) <= 1e-12
        assert strict_relerr(A.tvp_partial(xs[1:]), y_ref) <= 1e-12
        assert abs(A.tvp_full(xs) - a_ref) <= 1e-12 * (1 + abs(a_ref))


def test_block_small_vs_reference(small):
    for block, outer, Hm, xs, y_ref, a_ref in small["bhhb"]:
        T = P.BhhbTensor(len(block), block, outer, Hm)
        assert strict_relerr(T.tvp_partial(xs[1:]), y_ref) <= 1e-12
        assert abs(T.tvp_full(xs) - a_ref) <= 1e-12 * (1 + abs(a_ref))
    for m, C, xs, y_ref, a_ref in small["baab"]:
        T = P.BaabTensor(m, C)
        assert strict_relerr(T.tvp_partial(xs[1:]), y_ref) <= 1e-12
        assert abs(T.tvp_full(xs) - a_ref) <= 1e-12 * (1 + abs(a_ref))
    for levels, G, xs, y_ref, a_ref in small["levelk"]:
        T = P.LevelKHankelTensor(len(levels[0]), levels, G)
        assert strict_relerr(T.tvp_partial(xs[1:]), y_ref) <= 1e-12
        assert abs(T.tvp_full(xs) - a_ref) <= 1e-12 * (1 + abs(a_ref))


def test_times_matrices_small_vs_reference(small):
    for shape, h, mats, T_ref in small["times_matrices"]:
        T = P.times_matrices(P.HankelTensor(shape, h), mats)
        assert T.shape == T_ref.shape
        assert strict_relerr(T, T_ref) <= 1e-12


def test_bhhb_matrix_return_and_identities():
    rng = np.random.default_rng(6)
    T = P.BhhbTensor(3, (2, 3, 2), (3, 2, 2), rand_vec(rng, 25).reshape(5, 5))
    xs = [rand_vec(rng, 6), rand_vec(rng, 4)]
    Y = T.tvp_partial(xs, as_matrix=True)
    assert Y.shape == (2, 3)
    np.testing.assert_array_equal(P.vec(Y), T.tvp_partial(xs))
    # unit outer blocks reduce to the 1D Hankel tensor (tests/test_block.py:82-90)
    h = rand_vec(rng, 7)
    Tb = P.BhhbTensor(3, (3, 3, 3), (1, 1, 1), h[:, None])
    Hh = P.HankelTensor((3, 3, 3), h)
    xs = [rand_vec(rng, 3) for _ in range(2)]
    np.testing.assert_allclose(Tb.tvp_partial(xs), Hh.tvp_partial(xs), atol=1e-12)


# ---- random oracle equivalence (acceptance criteria 1 & 2) -----------------

def test_criterion1_random_hankel_vs_dense():
    rng = np.random.default_rng(101)
    worst = 0.0
    for _ in range(200):
        m = int(rng.integers(2, 5))
        shape = tuple(int(rng.integers(2, 8)) for _ in range(m))
        dof = sum(shape) - m + 1
        h = rand_vec(rng, dof)
        H = P.HankelTensor(shape, h)
        dense = O.dense_hankel(h, shape)
        xs = [rand_vec(rng, n) for n in shape]
        worst = max(worst, relerr(H.tvp_partial(xs[1:]), O.brute_tvp_partial(dense, xs[1:])))
        ref = O.brute_tvp_full(dense, xs)
        worst = max(worst, abs(H.tvp_full(xs) - ref) / (abs(ref) + 1.0))
    assert worst <= 1e-11


def test_criterion2_random_blocks_vs_dense():
    rng = np.random.default_rng(102)
    worst = 0.0
    for _ in range(40):
        m = int(rng.integers(2, 4))
        block = tuple(int(rng.integers(2, 5)) for _ in range(m))
        outer = tuple(int(rng.integers(2, 4)) for _ in range(m))
        d_in, d_out = sum(block) - m + 1, sum(outer) - m + 1
        Hm = rand_vec(rng, d_in * d_out).reshape(d_in, d_out)
        T = P.BhhbTensor(m, block, outer, Hm)
        dense = O.dense_bhhb(Hm, block, outer)
        xs = [rand_vec(rng, n) for n in T.mode_sizes]
        worst = max(worst, relerr(T.tvp_partial(xs[1:]), O.brute_tvp_partial(dense, xs[1:])))
    assert worst <= 1e-11


def test_every_supported_length():
    """One product per on-chip FFT length (powers of two and 3*2^k)."""
    rng = np.random.default_rng(7)
    for d in [1, 2, 3, 5, 8, 11, 16, 20, 24, 30, 40, 48, 60, 90, 96, 150, 190, 256, 300, 384,
              500, 700, 768, 1000, 1500, 1536, 2000, 3000, 3072, 4000, 4093, 5998, 6144, 8000]:
        # order-2 tensor with d_H = d: shape (n1, n2), n1 + n2 - 1 = d
        n1 = max(1, d // 3)
        n2 = d + 1 - n1
        h = rand_vec(rng, d)
        x = rand_vec(rng, n2)
        y = P.HankelTensor((n1, n2), h).tvp_partial([x])
        ref = O.hankel_tvp_partial(h, (n1, n2), [x])
        assert strict_relerr(y, ref) <= 1e-12, d


# ---- configs through the batched device API --------------------------------

def test_cfg1_real_inputs():
    g = load_golden("cfg1.npz")
    h, x = workloads.cfg1()
    dh = torch.from_numpy(h).cuda()[None]
    dx = torch.from_numpy(x).cuda()[None]
    y = batched.hankel_tvp_partial(dh, [dx, dx], (100,) * 3)[0].cpu().numpy()
    assert strict_relerr(y, g["y"]) <= TOL
    assert strict_relerr(y, g["y_dense"]) <= TOL
    a = batched.hankel_tvp_full(dh, [dx, dx, dx], (100,) * 3)[0].item()
    assert abs(a - complex(g["alpha"])) <= TOL * abs(complex(g["alpha"]))
    # drop-in object path
    H = P.HankelTensor((100,) * 3, h)
    assert strict_relerr(H.tvp_partial([x, x]), g["y"]) <= TOL
    assert abs(H.tvp_full([x, x, x]) - complex(g["alpha"])) <= TOL * abs(complex(g["alpha"]))


def test_cfg2_full_batch():
    g = load_golden("cfg2.npz")
    h, x = workloads.cfg2()
    dh = torch.from_numpy(h).cuda()
    dx = torch.from_numpy(x).cuda()
    y = batched.hankel_tvp_partial(dh, [dx, dx, dx], (1024,) * 4).cpu().numpy()
    # reference (exact L = 4093) golden outputs and per-product norms
    for k, b in enumerate(g["sel"]):
        assert strict_relerr(y[b], g["y"][k]) <= TOL
    norms = np.linalg.norm(y, axis=1)
    np.testing.assert_allclose(norms, g["norms"], rtol=TOL)
    np.testing.assert_allclose(y[:, 0], g["first"], rtol=1e-9, atol=1e-9 * np.abs(g["first"]).max())
    # every product against the oracle
    ref = O.hankel_tvp_partial_batch(h, [x, x, x], (1024,) * 4, length=4096)
    err = np.linalg.norm(y - ref, axis=1) / np.linalg.norm(ref, axis=1)
    assert err.max() <= TOL


def test_cfg2_mixed_vectors_and_cached_spectrum():
    rng = np.random.default_rng(22)
    B, n, m = 64, 1024, 4
    d = m * (n - 1) + 1
    h = rng.standard_normal((B, d)) + 1j * rng.standard_normal((B, d))
    xs = [rng.standard_normal((B, n)) + 1j * rng.standard_normal((B, n)) for _ in range(3)]
    dh = torch.from_numpy(h).cuda()
    dxs = [torch.from_numpy(v).cuda() for v in xs]
    y = batched.hankel_tvp_partial(dh, dxs, (n,) * m).cpu().numpy()
    ref = O.hankel_tvp_partial_batch(h, xs, (n,) * m, length=4096)
    assert strict_relerr(y, ref) <= TOL
    spec = batched.hankel_spectrum(dh, (n,) * m)
    y2 = batched.hankel_tvp_partial(spec, dxs, (n,) * m, spectrum=True).cpu().numpy()
    assert strict_relerr(y2, ref) <= TOL
    a = batched.hankel_tvp_full(spec, [dxs[0]] + dxs, (n,) * m, spectrum=True).cpu().numpy()
    a_ref = np.array([O.hankel_tvp_full(h[b], (n,) * m, [xs[0][b]] + [v[b] for v in xs])
                      for b in range(4)])
    assert strict_relerr(a[:4], a_ref) <= TOL


def test_cfg5_times_matrices_iteration():
    g = load_golden("cfg5.npz")
    sig, U0, shape = workloads.cfg5(signals=4)
    dh = torch.from_numpy(sig).cuda()
    dU = torch.from_numpy(np.ascontiguousarray(np.conj(U0))).cuda()[None].expand(4, -1, -1)
    dU = dU.contiguous()
    T = batched.times_matrices(dh, shape, [dU, dU]).cpu().numpy()
    assert strict_relerr(T[0][g["rows"]], g["T1_rows"]) <= TOL
    for s in range(4):
        ref = O.times_matrices_fast(sig[s], shape, [np.conj(U0)] * 2, length=6144)
        assert strict_relerr(T[s], ref) <= TOL


def test_lazy_conj_views_are_materialised():
    """x.conj().contiguous() of a contiguous CUDA tensor is a lazy view in torch;
    the batched API must pass the conjugated values, not the raw storage."""
    rng = np.random.default_rng(31)
    shape = (50, 60, 70)
    d = sum(shape) - 2
    h = rng.standard_normal((2, d)) + 1j * rng.standard_normal((2, d))
    x = rng.standard_normal((2, 60)) + 1j * rng.standard_normal((2, 60))
    z = rng.standard_normal((2, 70)) + 1j * rng.standard_normal((2, 70))
    dx = torch.from_numpy(x).cuda().conj().contiguous()
    assert dx.is_conj()
    y = batched.hankel_tvp_partial(torch.from_numpy(h).cuda(), [dx, torch.from_numpy(z).cuda()],
                                   shape).cpu().numpy()
    ref = np.stack([O.hankel_tvp_partial(h[b], shape, [np.conj(x[b]), z[b]]) for b in range(2)])
    assert strict_relerr(y, ref) <= TOL


def test_concurrent_numpy_calls_are_independent():
    """Several host threads share the per-device staging buffers of the
    numpy-facing path; every call must still return its own product
    (reference SPEC: deterministic results regardless of schedule)."""
    import threading

    rng = np.random.default_rng(31)
    cases = []
    for k in range(8):
        shape = (100 + k, 120, 120)
        h = rand_vec(rng, sum(shape) - 2)
        x = rand_vec(rng, 120)
        cases.append((P.HankelTensor(shape, h), x, O.hankel_tvp_partial(h, shape, [x, x])))
    errs = []

    def work(T, x, ref):
        for _ in range(20):
            y = T.tvp_partial([x, x])
            errs.append(strict_relerr(y, ref))

    ths = [threading.Thread(target=work, args=c) for c in cases]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    assert len(errs) == 160 and max(errs) <= 1e-12

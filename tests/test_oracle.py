"""Pin the CPU oracle to the reference (CPU-only; no GPU needed).

(a) known-answer vectors from the reference test-suite, (b) golden outputs
produced by the reference itself (oracle/gen_golden.py), (c) the oracle's FFT
path against its own dense brute force.
"""

import numpy as np
import pytest

from oracle import hankel_oracle as O
from paper_1401_6238_b200 import workloads
from tests.helpers import load_golden, load_small_cases, rand_vec, relerr, strict_relerr


# ---- (a) known answers (reference tests/test_hankel.py, test_block.py) ----

def test_counting_example():
    # tests/test_hankel.py:131-134
    y = O.hankel_tvp_partial(np.arange(7), (3, 3, 3), [np.ones(3)] * 2)
    np.testing.assert_allclose(y, [18, 27, 36], atol=1e-11)


def test_acirc_all_ones_full_product():
    # tests/test_hankel.py:79-81
    assert O.acirc_tvp_full([1, 2, 3], [np.ones(3)] * 3) == pytest.approx(54.0)


def test_spectrum_impulse_and_constant():
    # tests/test_hankel.py:16-23
    np.testing.assert_allclose(O.acirc_spectrum(np.eye(5)[0]), np.full(5, 0.2), atol=1e-14)
    np.testing.assert_allclose(O.acirc_spectrum(np.ones(4)), [1, 0, 0, 0], atol=1e-14)


def test_zero_generators():
    np.testing.assert_allclose(O.hankel_tvp_partial(np.zeros(7), (3, 3, 3), [np.ones(3)] * 2),
                               0, atol=1e-14)
    np.testing.assert_allclose(
        O.bhhb_tvp_partial(np.zeros((4, 4)), (2, 2, 2), (2, 2, 2), [np.ones(4)] * 2), 0,
        atol=1e-14)


def test_eigenpair_identity():
    # Corollary 2.2 via the fast product (tests/test_hankel.py:42-47)
    y = O.acirc_tvp_partial([1, 2, 3], [np.ones(3)] * 2)
    np.testing.assert_allclose(y, 18 * np.ones(3), atol=1e-12)


# ---- (b) golden outputs from the reference ---------------------------------

@pytest.fixture(scope="module")
def small():
    return load_small_cases()


def test_small_hankel_vs_reference(small):
    for shape, h, xs, y_ref, a_ref in small["hankel"]:
        assert strict_relerr(O.hankel_tvp_partial(h, shape, xs[1:]), y_ref) <= 1e-13
        assert abs(O.hankel_tvp_full(h, shape, xs) - a_ref) <= 1e-13 * (1 + abs(a_ref))


def test_small_acirc_vs_reference(small):
    for m, c, xs, spec_ref, y_ref, a_ref in small["acirc"]:
        np.testing.assert_allclose(O.acirc_spectrum(c), spec_ref, atol=1e-15, rtol=0)
        assert strict_relerr(O.acirc_tvp_partial(c, xs[1:]), y_ref) <= 1e-13
        assert abs(O.acirc_tvp_full(c, xs) - a_ref) <= 1e-13 * (1 + abs(a_ref))


def test_small_block_vs_reference(small):
    for block, outer, Hm, xs, y_ref, a_ref in small["bhhb"]:
        assert strict_relerr(O.bhhb_tvp_partial(Hm, block, outer, xs[1:]), y_ref) <= 1e-13
        assert abs(O.bhhb_tvp_full(Hm, block, outer, xs) - a_ref) <= 1e-13 * (1 + abs(a_ref))
    for m, C, xs, y_ref, a_ref in small["baab"]:
        assert strict_relerr(O.baab_tvp_partial(C, xs[1:]), y_ref) <= 1e-13
        assert abs(O.baab_tvp_full(C, xs) - a_ref) <= 1e-13 * (1 + abs(a_ref))
    for levels, G, xs, y_ref, a_ref in small["levelk"]:
        assert strict_relerr(O.levelk_tvp_partial(G, levels, xs[1:]), y_ref) <= 1e-13
        assert abs(O.levelk_tvp_full(G, levels, xs) - a_ref) <= 1e-13 * (1 + abs(a_ref))


def test_small_times_matrices_vs_reference(small):
    for shape, h, mats, T_ref in small["times_matrices"]:
        assert strict_relerr(O.times_matrices(h, shape, mats), T_ref) <= 1e-13
        assert strict_relerr(O.times_matrices_fast(h, shape, mats), T_ref) <= 1e-13


# ---- (c) oracle fast path vs its own dense brute force ----------------------

def test_oracle_fast_vs_dense_random():
    # acceptance criterion 1 shape (tests/test_acceptance.py:37-52)
    rng = np.random.default_rng(101)
    for _ in range(100):
        m = int(rng.integers(2, 5))
        shape = tuple(int(rng.integers(2, 8)) for _ in range(m))
        h = rand_vec(rng, sum(shape) - m + 1)
        dense = O.dense_hankel(h, shape)
        xs = [rand_vec(rng, n) for n in shape]
        assert relerr(O.hankel_tvp_partial(h, shape, xs[1:]),
                      O.brute_tvp_partial(dense, xs[1:])) <= 1e-11
        assert relerr(O.hankel_tvp_partial_padded(h, shape, xs[1:]),
                      O.brute_tvp_partial(dense, xs[1:])) <= 1e-11


def test_oracle_block_vs_dense():
    rng = np.random.default_rng(102)
    block, outer = (3, 2, 4), (2, 3, 2)
    Hm = rand_vec(rng, 7 * 5).reshape(7, 5)
    dense = O.dense_bhhb(Hm, block, outer)
    xs = [rand_vec(rng, b * o) for b, o in zip(block, outer)]
    assert relerr(O.bhhb_tvp_partial(Hm, block, outer, xs[1:]),
                  O.brute_tvp_partial(dense, xs[1:])) <= 1e-11
    C = rand_vec(rng, 12).reshape(3, 4)
    dense = O.dense_baab(C, 3)
    xs = [rand_vec(rng, 12) for _ in range(3)]
    assert relerr(O.baab_tvp_partial(C, xs[1:]), O.brute_tvp_partial(dense, xs[1:])) <= 1e-11


# ---- configs: oracle vs reference golden at full size -----------------------

def test_cfg1_golden():
    g = load_golden("cfg1.npz")
    h, x = workloads.cfg1()
    y = O.hankel_tvp_partial(h, (100,) * 3, [x, x])
    assert strict_relerr(y, g["y"]) <= 1e-14
    assert strict_relerr(g["y"], g["y_dense"]) <= 1e-12
    a = O.hankel_tvp_full(h, (100,) * 3, [x, x, x])
    assert abs(a - complex(g["alpha"])) <= 1e-12 * abs(complex(g["alpha"]))


def test_cfg2_golden_pow2_oracle():
    g = load_golden("cfg2.npz")
    h, x = workloads.cfg2()
    np.testing.assert_allclose(h.sum(axis=1)[:8], g["h_sum"], rtol=1e-15)
    y = O.hankel_tvp_partial_batch(h, [x, x, x], (1024,) * 4, length=4096)
    assert strict_relerr(y[g["sel"]], g["y"]) <= 1e-13
    np.testing.assert_allclose(np.linalg.norm(y, axis=1), g["norms"], rtol=1e-12)


def test_cfg4_golden():
    g = load_golden("cfg4.npz")
    H, X = workloads.cfg4()
    y = O.bhhb_tvp_partial_batch(H[g["sel"]], X[g["sel"]], (64,) * 3, (64,) * 3)
    assert strict_relerr(y, g["y"]) <= 1e-13


def test_cfg5_golden():
    g = load_golden("cfg5.npz")
    sig, U0, shape = workloads.cfg5(signals=1)
    np.testing.assert_allclose(U0, g["U0"], rtol=0, atol=1e-15)
    T1 = O.times_matrices_fast(sig[0], shape, [np.conj(U0)] * 2, length=6144)
    assert strict_relerr(T1[g["rows"]], g["T1_rows"]) <= 1e-12
    U1 = O.truncated_left_singular_vectors(T1.reshape(shape[0], -1), 5)
    P, Pref = U1 @ U1.conj().T, g["U1"] @ g["U1"].conj().T
    assert np.linalg.norm(P - Pref) <= 1e-10 * np.linalg.norm(Pref)


@pytest.mark.slow
def test_cfg3_golden_pow2_oracle():
    g = load_golden("cfg3.npz")
    h, x = workloads.cfg3()
    y = O.hankel_tvp_partial_padded(h, (1 << 22,) * 3, [x, x], length=1 << 24)
    assert strict_relerr(y[g["idx"]], g["y"]) <= 1e-12
    assert abs(np.linalg.norm(y) - float(g["norm"])) <= 1e-12 * float(g["norm"])

"""GPU public FFT wrappers (reference fourier.py) against numpy's pocketfft
and the reference tests/test_fourier.py known answers."""

import numpy as np
import pytest

import paper_1401_6238_b200 as P
from tests.helpers import rand_vec

pytestmark = pytest.mark.gpu


def test_impulse_constant_roundtrip():
    np.testing.assert_allclose(P.fft1([1, 0, 0, 0]), np.ones(4), atol=1e-14)
    np.testing.assert_allclose(P.fft1([1, 1, 1, 1]), [4, 0, 0, 0], atol=1e-14)
    rng = np.random.default_rng(0)
    v = rand_vec(rng, 7)
    np.testing.assert_allclose(P.ifft1(P.fft1(v)), v, rtol=1e-13, atol=1e-13)


def test_dft_matrix_all_small_lengths():
    # tests/test_fourier.py:30-38
    rng = np.random.default_rng(1)
    for n in range(1, 33):
        v = rand_vec(rng, n)
        F = P.fourier_matrix(n)
        np.testing.assert_allclose(P.fft1(v), F @ v, rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(P.ifft1(v), np.conj(F) @ v / n, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("n", [97, 4093, 5998, 6144, 10007])
def test_long_and_prime_lengths(n):
    rng = np.random.default_rng(n)
    v = rng.standard_normal((3, n)) + 1j * rng.standard_normal((3, n))
    ref = np.fft.fft(v)
    assert np.linalg.norm(P.fft1(v) - ref) <= 1e-12 * np.linalg.norm(ref)
    ref = np.fft.ifft(v)
    assert np.linalg.norm(P.ifft1(v) - ref) <= 1e-12 * np.linalg.norm(ref)


def test_fft2_fftn():
    rng = np.random.default_rng(3)
    M = rng.standard_normal((19, 30)) + 1j * rng.standard_normal((19, 30))
    assert np.linalg.norm(P.fft2(M) - np.fft.fft2(M)) <= 1e-12 * np.linalg.norm(np.fft.fft2(M))
    assert np.linalg.norm(P.ifft2(M) - np.fft.ifft2(M)) <= 1e-12 * np.linalg.norm(np.fft.ifft2(M))
    T = rng.standard_normal((5, 6, 7)) + 1j * rng.standard_normal((5, 6, 7))
    assert np.linalg.norm(P.fftn(T) - np.fft.fftn(T)) <= 1e-12 * np.linalg.norm(np.fft.fftn(T))
    assert np.linalg.norm(P.ifftn(T) - np.fft.ifftn(T)) <= 1e-12 * np.linalg.norm(np.fft.ifftn(T))


def test_block_spectra_match_numpy():
    """BhhbTensor / BaabTensor / LevelKHankelTensor .spectrum = ifft2 / ifftn of
    the generator (block.py:65-69, 125-127, 214-216)."""
    rng = np.random.default_rng(21)
    H = rng.standard_normal((9, 7)) + 1j * rng.standard_normal((9, 7))
    B = P.BhhbTensor(3, (3, 4, 4), (2, 3, 4), H)
    np.testing.assert_allclose(B.spectrum, np.fft.ifft2(H), rtol=0, atol=1e-13)
    C = rng.standard_normal((5, 6)) + 1j * rng.standard_normal((5, 6))
    np.testing.assert_allclose(P.BaabTensor(3, C).spectrum, np.fft.ifft2(C), rtol=0, atol=1e-13)
    levels = ((2, 3, 2), (3, 2, 2), (2, 2, 3))
    G = rng.standard_normal((5, 5, 5)) + 1j * rng.standard_normal((5, 5, 5))
    T = P.LevelKHankelTensor(3, levels, G)
    np.testing.assert_allclose(T.spectrum, np.fft.ifftn(G), rtol=0, atol=1e-13)

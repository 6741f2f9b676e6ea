"""Seeded synthetic inputs for the five BASELINE.json configurations.

Shapes, distributions and draw order follow SURVEY.md §8(d); every config k
draws from ``np.random.default_rng(k)``.  All inputs are synthetic by
definition (BASELINE.json "configs"); no dataset is involved.
"""

from __future__ import annotations

import numpy as np


def cfg1():
    """Order 3, n=100, float64: h[298], x[100] ~ N(0,1)."""
    rng = np.random.default_rng(1)
    h = rng.standard_normal(298)
    x = rng.standard_normal(100)
    return h, x


def cfg2(batch=4096, n=1024, m=4):
    """4096 independent order-4 n=1024 complex Hankel tensors, one x each."""
    rng = np.random.default_rng(2)
    d = m * (n - 1) + 1
    h = rng.standard_normal((batch, d)) + 1j * rng.standard_normal((batch, d))
    x = rng.standard_normal((batch, n)) + 1j * rng.standard_normal((batch, n))
    return h, x


def cfg3(n=1 << 22, m=3):
    """One order-3 real tensor, n=2^22: h ~ N(0,1) (length 12,582,910), x ~ U[-1,1]."""
    rng = np.random.default_rng(3)
    h = rng.standard_normal(m * (n - 1) + 1)
    x = rng.uniform(-1.0, 1.0, n)
    return h, x


def cfg4(batch=1024, n=64, N=64, m=3):
    """BHHB order 3, blocks 64x64 -> H 190x190 complex; X (64x64) with x = vec(X)."""
    rng = np.random.default_rng(4)
    din, dout = m * (n - 1) + 1, m * (N - 1) + 1
    H = rng.standard_normal((batch, din, dout)) + 1j * rng.standard_normal((batch, din, dout))
    X = rng.standard_normal((batch, n, N)) + 1j * rng.standard_normal((batch, n, N))
    return H, X


def cfg5(signals=256, n_samples=5998, K=5, snr_db=20.0, rank=5, n=2000):
    """Damped complex exponentials + 20 dB noise; shared U0 for the HOOI loop.

    Per signal: dampings U[0.001,0.05], frequencies U[0,1), phases U[0,2pi),
    c_k = exp(i phi_k), z_k = exp(-alpha_k + 2 pi i f_k) (the ExpModel1D
    convention, reference expfit.py:64-70, dt=1), noise sigma/sqrt(2)(N+iN)
    (expfit.py:30-33) with sigma^2 = mean|x|^2 / 10^(snr/10).
    U0 = fix_phase(qr(N + iN).Q) of shape (n, rank) is drawn FIRST, so any
    prefix of the signal batch (signals=s) sees the same U0 and signals.
    """
    rng = np.random.default_rng(5)
    Q, _ = np.linalg.qr(rng.standard_normal((n, rank)) + 1j * rng.standard_normal((n, rank)))
    U0 = _fix_phase(Q)
    t = np.arange(n_samples)
    sig = np.empty((signals, n_samples), dtype=np.complex128)
    for s in range(signals):
        damp = rng.uniform(0.001, 0.05, K)
        freq = rng.uniform(0.0, 1.0, K)
        phase = rng.uniform(0.0, 2 * np.pi, K)
        c = np.exp(1j * phase)
        z = np.exp(-damp + 2j * np.pi * freq)
        x = (c[None, :] * z[None, :] ** t[:, None]).sum(axis=1)
        sigma = np.sqrt(np.mean(np.abs(x) ** 2) / 10 ** (snr_db / 10))
        noise = sigma / np.sqrt(2.0) * (rng.standard_normal(n_samples)
                                        + 1j * rng.standard_normal(n_samples))
        sig[s] = x + noise
    shape = (n, n, n)
    return sig, U0, shape


def _fix_phase(U):
    """Largest-|.| entry of each column real positive (reference decompose.py:23-32)."""
    U = np.array(U, dtype=np.complex128, copy=True)
    idx = np.argmax(np.abs(U), axis=0)
    a = U[idx, np.arange(U.shape[1])]
    scale = np.where(np.abs(a) > 0, np.conj(a) / np.where(np.abs(a) > 0, np.abs(a), 1), 1)
    return U * scale[None, :]


def tm_large_inputs():
    """Seeded inputs of the two-level times_matrices parity cases
    (oracle/gen_golden_r2.py, tests/test_gpu_tm_large.py): order 3 with n = 3000
    (d_H = 8998) and r = 3, and order 2 (5000, 4000) with r = 2."""
    rng = np.random.default_rng(777)

    def rv(n):
        return rng.standard_normal(n) + 1j * rng.standard_normal(n)

    h3 = rv(8998)
    M3 = rv(3000 * 3).reshape(3000, 3)
    M3b = rv(3000 * 3).reshape(3000, 3)
    h2 = rv(8999)
    M2 = rv(4000 * 2).reshape(4000, 2)
    return h3, M3, M3b, h2, M2

"""Discrete Fourier transforms with the reference's pinned normalisation
(forward unnormalised, inverse 1/n per axis; reference fourier.py:1-49),
computed on the GPU for ANY length.

Each length-n transform is a Bluestein chirp transform written as an order-2
Hankel product, so it runs on the same fused kernels as the tensor products:
with chi_s = exp(-i pi s^2 / n) (s^2 taken mod 2n exactly),
    fft(v)_k = conj(chi_k) * sum_j chi_{j+k} * (v_j conj(chi_j)),
i.e. y = H x with H the n x n Hankel matrix of generating vector
chi[0 .. 2n-2].  The chirp spectrum is computed once per (n, device) and
broadcast over the batch (batch stride 0); inverse transforms use
ifft(v) = conj(fft(conj(v))) / n.
"""

from __future__ import annotations

import numpy as np
import torch

from . import batched
from ._device import require_cuda


def _as_complex(a) -> np.ndarray:
    return np.asarray(a, dtype=np.complex128)


def _check_nonempty(a):
    """fourier.py:22-25."""
    if a.size == 0:
        raise ValueError("empty input")
    return a


def fourier_matrix(n: int) -> np.ndarray:
    """The n-by-n matrix (exp(-2 pi i j k / n))_{j,k} (fourier.py:14-19)."""
    if n < 1:
        raise ValueError("size must be positive")
    jk = np.outer(np.arange(n), np.arange(n))
    return np.exp(-2j * np.pi * jk / n)


_chirps: dict = {}


def _chirp(n: int, dev: int):
    key = (n, dev)
    c = _chirps.get(key)
    if c is None:
        s = np.arange(2 * n - 1, dtype=np.int64)
        chi = np.exp(-1j * np.pi * ((s * s) % (2 * n)) / n)
        dchi = torch.from_numpy(chi).to(f"cuda:{dev}")
        spec = batched.hankel_spectrum(dchi[None], (n, n))
        c = (dchi[:n].clone(), spec)
        _chirps[key] = c
    return c


def _fft_last_axis(x: torch.Tensor, inverse: bool) -> torch.Tensor:
    """Batched transform of a (B, n) complex128 device tensor along axis 1."""
    B, n = x.shape
    dev = x.device.index
    chi, spec = _chirp(n, dev)
    if inverse:
        x = torch.conj_physical(x)
    u = (x * torch.conj_physical(chi)[None, :]).contiguous()
    y = batched.hankel_tvp_partial(spec.expand(B, -1), [u], (n, n), spectrum=True)
    y = y * torch.conj_physical(chi)[None, :]
    if inverse:
        y = torch.conj_physical(y) / n
    return y


def _transform(a, axes, inverse: bool) -> np.ndarray:
    a = _check_nonempty(_as_complex(a))
    dev = require_cuda()
    t = torch.from_numpy(np.ascontiguousarray(a)).to(f"cuda:{dev}")
    for ax in axes:
        moved = torch.movedim(t, ax, -1).contiguous()
        shp = moved.shape
        y = _fft_last_axis(moved.reshape(-1, shp[-1]), inverse)
        t = torch.movedim(y.reshape(shp), -1, ax)
    return t.cpu().numpy()


def fft1(v) -> np.ndarray:
    """np.fft.fft (fourier.py:28-29): last axis."""
    return _transform(v, [-1], False)


def ifft1(v) -> np.ndarray:
    """np.fft.ifft (fourier.py:32-33): last axis, 1/n."""
    return _transform(v, [-1], True)


def fft2(M) -> np.ndarray:
    """np.fft.fft2 (fourier.py:36-37): last two axes."""
    M = _as_complex(M)
    return _transform(M, [-1, -2], False)


def ifft2(M) -> np.ndarray:
    """np.fft.ifft2 (fourier.py:40-41)."""
    M = _as_complex(M)
    return _transform(M, [-1, -2], True)


def fftn(T) -> np.ndarray:
    """np.fft.fftn (fourier.py:44-45): all axes."""
    T = _as_complex(T)
    return _transform(T, list(range(T.ndim)), False)


def ifftn(T) -> np.ndarray:
    """np.fft.ifftn (fourier.py:48-49)."""
    T = _as_complex(T)
    return _transform(T, list(range(T.ndim)), True)

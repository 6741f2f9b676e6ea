"""GPU HOOI driver loop against the reference's own
iterates (golden cfg5 U1, U2) and an oracle restatement of
decompose.py:142-184."""

import numpy as np
import pytest
import torch

import paper_1401_6238_b200 as P
from oracle import hankel_oracle as O
from paper_1401_6238_b200 import workloads
from paper_1401_6238_b200.hooi import hooi_symmetric, hooi_symmetric_batched
from tests.helpers import load_golden

pytestmark = pytest.mark.gpu


def _proj_err(U, Uref):
    P1, P2 = U @ U.conj().T, Uref @ Uref.conj().T
    return np.linalg.norm(P1 - P2) / np.linalg.norm(P2)


def test_cfg5_two_sweeps_match_reference_iterates():
    g = load_golden("cfg5.npz")
    sig, U0, shape = workloads.cfg5(signals=2)
    dh = torch.from_numpy(sig).cuda()
    dU0 = torch.from_numpy(U0).cuda()
    U1 = hooi_symmetric_batched(dh, shape, 5, dU0, max_iter=1)[0].cpu().numpy()
    U2 = hooi_symmetric_batched(dh, shape, 5, dU0, max_iter=2)[0].cpu().numpy()
    assert _proj_err(U1, g["U1"]) <= 1e-10
    assert _proj_err(U2, g["U2"]) <= 1e-10
    # columns (phase-fixed) agree where singular values are separated
    assert np.linalg.norm(U1 - g["U1"]) <= 1e-8 * np.linalg.norm(g["U1"])


def _oracle_hooi(h, shape, rank, tol, max_iter):
    """Restatement of decompose.py:142-184 on the CPU oracle."""
    n, m = shape[0], len(shape)
    red = np.asarray(h)[np.add.outer(np.arange(n), np.arange(len(h) - n + 1))]
    U = O.truncated_left_singular_vectors(red, rank)

    def core_with(Um):
        T = O.times_matrices_fast(h, shape, [np.conj(Um)] * (m - 1))
        S = np.tensordot(T, np.conj(Um), axes=([0], [0]))
        return T, np.moveaxis(S, -1, 0)

    T, S = core_with(U)
    fits = [float(np.linalg.norm(S))]
    for _ in range(max_iter):
        U = O.truncated_left_singular_vectors(T.reshape(n, -1), rank)
        T, S = core_with(U)
        fits.append(float(np.linalg.norm(S)))
        if abs(fits[-1] - fits[-2]) / max(fits[-1], np.finfo(float).eps) < tol:
            break
    return U, fits


def test_hooi_symmetric_dropin_matches_oracle():
    # exact rank-2 damped exponentials (reference tests/test_decompose.py style)
    n = 40
    t = np.arange(3 * n - 2)
    z = np.exp(np.array([-0.01 + 0.7j, -0.02 + 2.1j]))
    h = (np.array([1.0, 0.5j])[None, :] * z[None, :] ** t[:, None]).sum(axis=1)
    H = P.HankelTensor((n,) * 3, h)
    res = hooi_symmetric(H, 2, tol=1e-12, max_iter=20)
    U_ref, fits_ref = _oracle_hooi(h, (n,) * 3, 2, 1e-12, 20)
    assert _proj_err(res.factor, U_ref) <= 1e-10
    assert abs(res.fits[-1] - fits_ref[-1]) <= 1e-10 * fits_ref[-1]
    assert res.core.shape == (2, 2, 2)
    assert res.monotone
